"""Per-step cost factors of bench.py: L2 flush and clock samplers (each
configuration from a fresh engine: identical iterations)."""
import subprocess, sys, threading
sys.path.insert(0, '/root/repo')
import torch, scenes
import paper_1403_0240_b200 as P
sc = scenes.cfg2()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

def run(k, do_flush, sampler):
    eng = P.RegionCompetition(sc.image, sc.labels, P.EnergyConfig("ps", "poisson", smooth_radius=4),
                              P.SobolevParams(6.0), P.OptimizerConfig("sobolev", vanish_grace=5))
    stream = torch.cuda.ExternalStream(eng.stream)
    for _ in range(3):
        eng.iterate()
    stop = threading.Event()
    def smi():
        while not stop.is_set():
            subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader"], capture_output=True)
            stop.wait(0.2)
    def nvml():
        import pynvml
        pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
        while not stop.is_set():
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            stop.wait(0.1)
    if sampler:
        threading.Thread(target=smi if sampler == "smi" else nvml, daemon=True).start()
    tot = 0.0
    for _ in range(k):
        if do_flush:
            flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream); eng.iterate(); e1.record(stream); e1.synchronize()
        tot += e0.elapsed_time(e1)
    stop.set()
    return tot / k

for do_flush, sampler in ((False, None), (True, None), (False, "smi"), (True, "smi"), (False, "nvml"), (True, "nvml"), (False, None)):
    print("flush", do_flush, "sampler", sampler, "ms/step", round(run(6, do_flush, sampler), 3), flush=True)
