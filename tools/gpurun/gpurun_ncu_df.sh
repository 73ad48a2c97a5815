#!/bin/bash
# ncu --set full + source page of k_accept_df at cfg4 iteration 20
python tools/profile_window.py --config cfg4 --warm 19 --iters 1 > gpurun_out/pw.log 2>&1 || { tail -5 gpurun_out/pw.log; exit 1; }
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_accept_df -c 1 -f -o gpurun_out/df_cfg4 python tools/profile_window.py --config cfg4 --warm 19 --iters 1 > gpurun_out/ncu_df.log 2>&1
tail -3 gpurun_out/ncu_df.log
ncu -i gpurun_out/df_cfg4.ncu-rep --page source --csv --print-source cuda > gpurun_out/df_cfg4_src.csv 2>/dev/null
ncu -i gpurun_out/df_cfg4.ncu-rep --page details --csv > gpurun_out/df_cfg4_details.csv 2>/dev/null
ls -la gpurun_out/df_cfg4*
