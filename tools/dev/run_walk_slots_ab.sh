O=gpurun_out/walk_slots_ab; mkdir -p $O
for i in 1 2; do for v in 1 0; do LMS_GZ_WALK_SLOTS=$v python bench.py --no-cpu --steps 3 > $O/bench_slots${v}_$i.log 2>&1; done; done
