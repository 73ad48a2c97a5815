#!/bin/bash
# ncu --set full of one kernel ($1 regex) at cfg4 iteration $2 (default 20); outputs gpurun_out/k_$3.*
K=$1; IT=${2:-20}; TAG=${3:-k}
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$K -c 1 -f -o gpurun_out/k_$TAG python tools/profile_window.py --config cfg4 --warm $((IT-1)) --iters 1 > gpurun_out/ncu_k.log 2>&1
tail -2 gpurun_out/ncu_k.log
ncu -i gpurun_out/k_$TAG.ncu-rep --page details --csv > gpurun_out/k_${TAG}_details.csv 2>/dev/null
ncu -i gpurun_out/k_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/k_${TAG}_src.csv 2>/dev/null
ls -la gpurun_out/k_$TAG*
