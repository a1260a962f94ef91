O=gpurun_out/jobs_in_flight; mkdir -p $O
for i in 1 2; do for n in 3 4; do python bench.py --no-cpu --steps 3 --jobs-in-flight $n > $O/bench_nj${n}_$i.log 2>&1; done; done
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1
