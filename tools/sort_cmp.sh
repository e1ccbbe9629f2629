L=$PWD/paper_0904_3151_b200/_native
for v in libepsgraph_b200 libeg_lb4 libeg_lb4m3 libeg_lb2m4 libeg_lb4i8; do
  echo "-- $v"; for m in 2480000 200000000 1400000000; do EG_LIB_PATH=$L/$v.so python tools/sort_bench.py $m 4000000 2>&1 | grep "path=0"; done
done
