# ncu evidence on the final kernel source: one --set full capture of k_sweep_gz
# (C4, original) and the bench command's launch list
O=gpurun_out/ncu_final; mkdir -p $O
python bench.py --steps 2 --warmup 3 --no-cpu > $O/bench_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_gz -s 1 -c 1 -o $O/gz_final \
  python tools/prof_one.py --schedule gz --sweeps 1 --reps 2 > $O/ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch.log 2>&1
