O=gpurun_out/tw6; mkdir -p $O
for i in 1 2; do python bench.py --no-cpu > $O/bench_walk_$i.log 2>&1; LMS_GZ_TILE_BFS=0 python bench.py --no-cpu > $O/bench_sort_$i.log 2>&1; done
