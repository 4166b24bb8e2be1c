# persistent FOM: sources unrolled per tile loop (rebuilds fom_persistent.o on the box)
for u in 4 6 8 12; do
  (cd paper_2103_01983_b200/csrc && touch fom_persistent.cu && make EXTRA=-DPTROM_FOM_UNR=$u > /dev/null 2>&1)
  echo "unr=$u"
  python tools/fom_time_probe.py 2>&1 | tail -1
done
(cd paper_2103_01983_b200/csrc && touch fom_persistent.cu && make > /dev/null 2>&1)
