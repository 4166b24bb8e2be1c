# hyperpair engine kernel: cache hints on the list and position loads (rebuilds rom.o on the box)
for h in 0 1 2 3; do
  (cd paper_2103_01983_b200/csrc && touch rom.cu && make EXTRA=-DPTROM_HP_HINT=$h > /dev/null 2>&1)
  echo "hint=$h"
  python tools/sweep_hp.py 512 1 0 2>&1 | tail -2
done
(cd paper_2103_01983_b200/csrc && touch rom.cu && make > /dev/null 2>&1)
