"""Measured compute peaks for the roofline denominators -> profiles/<tag>_peaks.json.

FFMA from scripts/ubench/peaks.cu (compiled here with nvcc); dense TF32 and
bf16 tensor-core GEMM throughput through cuBLAS (torch.matmul, 8192^3, median
of 10 after warm-up); HBM copy bandwidth (a 4 GiB device-to-device copy)."""
import json
import subprocess
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
exe = ROOT / "scripts" / "ubench" / "peaks"
subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(exe),
                str(ROOT / "scripts" / "ubench" / "peaks.cu")], check=True)
out = json.loads(subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout)


def gemm_tflops(dtype, tf32):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    n = 8192
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return 2 * n ** 3 / (ts[len(ts) // 2] * 1e-3) / 1e12


out["tf32_tflops_cublas"] = round(gemm_tflops(torch.float32, True), 1)
out["fp32_sgemm_tflops_cublas"] = round(gemm_tflops(torch.float32, False), 1)
out["bf16_tflops_cublas"] = round(gemm_tflops(torch.bfloat16, False), 1)
x = torch.empty(1 << 30, dtype=torch.float32, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    y.copy_(x)
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    y.copy_(x)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
out["hbm_copy_gbs"] = round(2 * x.numel() * 4 / (ts[len(ts) // 2] * 1e-3) / 1e9, 1)
out["gpu"] = torch.cuda.get_device_name()
(ROOT / "profiles").mkdir(exist_ok=True)
(ROOT / "profiles" / f"{tag}_peaks.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out))
