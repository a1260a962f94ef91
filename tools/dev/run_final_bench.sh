O=gpurun_out/final_r2d; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python bench.py > $O/bench.log 2>&1
LMS_LIB_PATH=$PWD/paper_1606_00803_b200/liblms_bounds.so timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests_bounds.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.log 2>&1
