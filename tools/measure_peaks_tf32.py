"""TF32 (and bf16, for the same-box ratio) tensor peak, measured like
MEASURED_PEAKS.json's bf16 figure: torch.matmul 8192^3 (2*N^3 flops), best of
10 (burst) and back to back for 4 s (sustained), CUDA events. Writes
profiles/r02_tf32_peak.json (the denominator of the fp32x3 / tf32 rooflines)."""
import json
import os
import sys
import time

import torch

N = 8192


def rate(dtype, tf32):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.backends.cudnn.allow_tf32 = tf32
    a = torch.randn(N, N, device="cuda", dtype=dtype)
    b = torch.randn(N, N, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.time()
    while time.time() - t0 < 4.0:
        for _ in range(20):
            a @ b
        n += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    fl = 2.0 * N ** 3
    return fl / (best / 1e3) / 1e12, fl * n / (e0.elapsed_time(e1) / 1e3) / 1e12


def main():
    tf_b, tf_s = rate(torch.float32, True)
    bf_b, bf_s = rate(torch.bfloat16, False)
    out = {"tf32_tflops": tf_b, "tf32_tflops_sustained": tf_s, "bf16_tflops_same_box": bf_b,
           "bf16_tflops_sustained_same_box": bf_s, "gpu": torch.cuda.get_device_name(0),
           "how": "torch.matmul fp32 with allow_tf32 (cuBLAS TF32 tensor cores) 8192^3, 2*N^3 flops: best of 10 "
                  "(burst) and back to back for 4 s (sustained), CUDA events; bf16 the same way for the ratio",
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                               "r02_tf32_peak.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
