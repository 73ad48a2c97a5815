python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/sweep_bench.py --points 1e6,1e7,1e8 --widths 1,2,4 --reps 5
timeout 300 python tools/config_run.py --config cfg4 --iters 26 > gpurun_out/pk_cfg4.txt 2>&1; tail -1 gpurun_out/pk_cfg4.txt | cut -c1-150
