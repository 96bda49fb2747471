"""Box probe: FP64 DGEMM peak (cuBLAS, for the roofline denominator only), HBM copy, host cores."""
import json, os, time, subprocess
import torch

def dgemm_peak(n=8192, reps=10):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); torch.matmul(a, b); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    burst = 2 * n**3 / best / 1e12
    # sustained 4 s
    t0 = time.time(); cnt = 0
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b); cnt += 1
        if cnt % 4 == 0: torch.cuda.synchronize()
    e.record(); e.synchronize()
    sus = 2 * n**3 * cnt / (s.elapsed_time(e) / 1e3) / 1e12
    return burst, sus

def hbm():
    x = torch.empty(1 << 28, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
    for _ in range(3): y.copy_(x)
    torch.cuda.synchronize(); best = 1e9
    for _ in range(10):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); y.copy_(x); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e) / 1e3)
    return 2 * x.numel() * 8 / best / 1e9

out = {}
out["host_cores"] = len(os.sched_getaffinity(0))
out["cpu_model"] = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].split(":")[1].strip()
try:
    import numba; out["numba"] = numba.__version__
except Exception as ex:
    out["numba"] = repr(ex)
out["gpu"] = torch.cuda.get_device_name(0)
p = torch.cuda.get_device_properties(0)
out["sms"] = p.multi_processor_count
out["dgemm_tflops_burst"], out["dgemm_tflops_sustained"] = dgemm_peak()
out["hbm_copy_gbs"] = hbm()
out["smi"] = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw", "--format=csv"], capture_output=True, text=True).stdout
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
