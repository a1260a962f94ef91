# ncu --set full of the GZ records kernel (C4 schedule build)
O=gpurun_out/ncu_rec; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gzd_records -c 1 -o $O/records \
  python tools/prof_one.py --schedule gz --sweeps 1 --reps 1 > $O/ncu.log 2>&1
