set -u
O=gpurun_out/tw1; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gz_build.py -x -q > $O/test_build.log 2>&1; echo "tests rc=$?" >> $O/test_build.log
for v in 1 0; do LMS_GZ_TILE_BFS=$v LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_e2e.py --steps 3 > $O/phases_$v.log 2>&1; done
timeout 600 python bench.py > $O/bench.log 2>&1
