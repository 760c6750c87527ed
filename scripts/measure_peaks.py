"""TF32 and FP32-FFMA tensor/FMA peaks on this B200, measured the way the
driver measures MEASURED_PEAKS.json's bf16 figure: cuBLAS GEMM 8192^3
(2*N^3 FLOP), best of 10 (burst) and back to back for 4 s (sustained), with
nvidia-smi clocks sampled during the sustained loop. TF32 = fp32 storage with
allow_tf32 (cuBLAS tf32 tensor cores); FFMA = fp32 with tf32 disabled.
    python scripts/measure_peaks.py > profiles/r02_measured_peaks_tf32_ffma.json"""
import json
import subprocess
import tempfile
import time

import torch

N = 8192


def measure(tf32):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.backends.cuda.matmul.fp32_precision = "tf32" if tf32 else "ieee"
    a = torch.randn(N, N, device="cuda")
    b = torch.randn(N, N, device="cuda")
    c = torch.empty(N, N, device="cuda")
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    burst = []
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=c)
        e.record()
        e.synchronize()
        burst.append(2 * N ** 3 / (s.elapsed_time(e) * 1e-3) / 1e12)
    path = tempfile.mktemp(suffix=".csv")
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "100"], stdout=open(path, "w"))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 0
    t0 = time.time()
    s.record()
    while time.time() - t0 < 4.0:
        for _ in range(10):
            torch.matmul(a, b, out=c)
        reps += 10
        torch.cuda.synchronize()
    e.record()
    e.synchronize()
    smi.terminate()
    smi.wait()
    sustained = reps * 2 * N ** 3 / (s.elapsed_time(e) * 1e-3) / 1e12
    clocks = [ln.split(",")[0].strip() for ln in open(path) if ln.strip()]
    mhz = sorted(float(x) for x in clocks if x.replace(".", "").isdigit())
    return max(burst), sustained, (mhz[len(mhz) // 2] if mhz else None)


tb, ts, tm = measure(True)
fb, fs, fm = measure(False)
print(json.dumps({
    "tf32_tflops": round(tb, 1), "tf32_tflops_sustained": round(ts, 1), "tf32_sm_mhz_median": tm,
    "fp32_tflops": round(fb, 2), "fp32_tflops_sustained": round(fs, 2), "fp32_sm_mhz_median": fm,
    "gpu": torch.cuda.get_device_name(), "torch": torch.__version__,
    "how": "cuBLAS torch.matmul fp32 8192^3, allow_tf32 on (tf32) / off (fp32 FFMA); best of 10 "
           "(burst) and back to back for 4 s (sustained), CUDA events"}, indent=1))
