python -m pytest tests/test_gpu_sweep.py tests/test_gpu_parity.py -q -x -k "sweep or site_kernel or sobolev" 2>&1 | tail -2
for m in bulk lsu; do RCB_K6_SITE=$m timeout 300 python tools/sweep_bench.py --points 1e6,1e7,1e8 --widths 1 --reps 5 | sed "s/^/$m /"; done
