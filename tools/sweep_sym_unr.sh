# fp64 unordered-pair velocity: sub-step unroll sweep (rebuilds allpairs_sym.o on the box)
for u in 4 8 16 32; do
  (cd paper_2103_01983_b200/csrc && touch allpairs_sym.cu && make EXTRA=-DPTROM_SYM_UNR=$u > /dev/null 2>&1)
  echo "unr=$u"
  bash tools/sweep_sym.sh
done
(cd paper_2103_01983_b200/csrc && touch allpairs_sym.cu && make > /dev/null 2>&1)
