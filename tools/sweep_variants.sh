# times alternative builds of libptrom_b200.so (tools/variants/*.so) on config 2 and config 5
for v in tools/variants/*.so; do
  cp paper_2103_01983_b200/libptrom_b200.so /tmp/lib_keep.so
  cp $v paper_2103_01983_b200/libptrom_b200.so
  echo "$v"; bash tools/sweep_sym.sh
  cp /tmp/lib_keep.so paper_2103_01983_b200/libptrom_b200.so
done
