#!/bin/bash
# Final measurement set: GPU tests, both bench arms, launch list and DRAM traffic of the
# bench window, ncu --set full of the top kernels.  Outputs under gpurun_out/final_*.
T=${TAG:-r02b}
python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest_gpu.log 2>&1; tail -2 gpurun_out/final_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee -a gpurun_out/final_pytest_gpu.log
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; cut -c1-300 gpurun_out/final_bench_ref.json
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err || tail -5 gpurun_out/final_bench.err
python -c "
import json;d=json.load(open('gpurun_out/final_bench.json'));print('cfg4',round(d['value']/1e9,3),'G/s',round(d['ms_per_step'],2),'ms e2e',round(d['e2e']['value']/1e9,3),d['phase_ms_per_iteration'], 'roof', round(d['roofline']['frac'],4))"
# launch list + DRAM bytes of every kernel over the bench window (iterations 6-25)
ncu --profile-from-start off --clock-control none --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --log-file gpurun_out/final_launches_cfg4.csv python tools/profile_window.py --config cfg4 --warm 5 --iters 20 > gpurun_out/final_ncu_w.log 2>&1; tail -1 gpurun_out/final_ncu_w.log
# ncu --set full of the top kernels at iteration 25
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:'k_accept_df|k_delta_ps_rec|k_fields_band3d_int|k_sobolev_pk' -f -o gpurun_out/final_full_cfg4 python tools/profile_window.py --config cfg4 --warm 24 --iters 1 > gpurun_out/final_ncu_full.log 2>&1; tail -1 gpurun_out/final_ncu_full.log
ncu -i gpurun_out/final_full_cfg4.ncu-rep --page details --csv > gpurun_out/final_ncu_full_cfg4.csv 2>/dev/null
# cfg2 launch list (10 iterations)
ncu --profile-from-start off --clock-control none --csv --metrics gpu__time_duration.sum --log-file gpurun_out/final_launches_cfg2.csv python tools/profile_window.py --config cfg2 --warm 5 --iters 10 > gpurun_out/final_ncu_c2.log 2>&1; tail -1 gpurun_out/final_ncu_c2.log
ls -la gpurun_out/final_*
