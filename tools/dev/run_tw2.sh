O=gpurun_out/tw2; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_gz_build.py -q > $O/test_build.log 2>&1
