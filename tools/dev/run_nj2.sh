O=gpurun_out/nj2; mkdir -p $O
for i in 1 2; do for n in 3 4; do LMS_CACHE_GB=64 python bench.py --no-cpu --steps 3 --jobs-in-flight $n > $O/bench_c64_nj${n}_$i.log 2>&1; done; done
