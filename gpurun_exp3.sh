python -m pytest tests/test_gpu_fp32.py -q 2>&1 | grep -E "AssertionError: \(|passed|failed" | head -10
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -k "ps_l2 or l2" 2>&1 | tail -2
timeout 900 python tools/ps_l2_probe.py --config cfg4 --sobolev 30 --l2 2 > gpurun_out/ps_l2_probe.txt 2>&1; tail -5 gpurun_out/ps_l2_probe.txt
RCB_ALLOC_LOG=1 timeout 600 python tools/alloc_probe.py > gpurun_out/alloc_probe2.json 2> gpurun_out/alloc_probe2.err; cat gpurun_out/alloc_probe2.json
