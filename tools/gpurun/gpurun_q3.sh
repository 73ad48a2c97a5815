#!/bin/bash
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_sweep.py -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
python bench.py --no-cpu-baseline --no-fp32 --no-full-run --no-sweep > gpurun_out/bq.json 2>gpurun_out/bq.err || tail -5 gpurun_out/bq.err
python -c "
import json;d=json.load(open('gpurun_out/bq.json'));print('cfg4',round(d['value']/1e9,3),'G/s',round(d['ms_per_step'],2),'ms',d['phase_ms_per_iteration'])
c=d.get('cfg2');print('cfg2',c and (round(c['iterations_per_s'],1), c['phase_ms_per_iteration']))"
for m in bulk lsu; do RCB_K6_SITE=$m timeout 300 python tools/sweep_bench.py --points 1e6,1e7,1e8 --widths 1 --reps 5 | sed "s/^/$m /"; done
