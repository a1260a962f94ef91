O=gpurun_out/tw10; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_gz_build.py -q > $O/test_build.log 2>&1
LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_e2e.py --steps 3 > $O/phases_1.log 2>&1
python bench.py --no-cpu > $O/bench.log 2>&1
