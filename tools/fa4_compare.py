"""Calibration for the fused attention kernel: time public Blackwell attention
forward kernels (library code, NOT on the product path) on attn_big's shape
(1 x 32 heads x 4096 x 4096, d = 128, bf16, non-causal) with CUDA events, so
the fused kernel's %-of-peak can be read against what the state of the art
reaches on the same box. Prints one JSON line per library that runs.

    python tools/fa4_compare.py [iters] [q/k multiplier]
"""
import json
import sys
import time

import torch

B, S, H, D = 1, 4096, 32, 128
FLOP = 4.0 * B * H * S * S * D
it = int(sys.argv[1]) if len(sys.argv) > 1 else 50


def timeit(fn, reps=20):
    """median over `it` samples of (events around `reps` back-to-back calls) / reps:
    amortises the Python launch path, which is slower than the kernel."""
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(max(3, it // 5)):
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / reps)
    ts.sort()
    return ts[len(ts) // 2], ts[0]


def main():
    torch.manual_seed(0)
    q = torch.randn(B, S, H, D, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(B, S, H, D, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(B, S, H, D, device="cuda", dtype=torch.bfloat16)
    if len(sys.argv) > 2:  # logit scale: integer-stream-like logits (~1e3) force O rescales
        q.mul_(float(sys.argv[2]))
        k.mul_(float(sys.argv[2]))
    ref = torch.nn.functional.scaled_dot_product_attention(q.transpose(1, 2).float(), k.transpose(1, 2).float(),
                                                           v.transpose(1, 2).float()).transpose(1, 2)
    cands = []
    try:
        from vllm.vllm_flash_attn.cute.interface import flash_attn_func as fa4
        cands.append(("vllm_flash_attn.cute (FA4, flash_fwd_sm100)", lambda: fa4(q, k, v)))
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"lib": "fa4", "unavailable": repr(e)[:300]}), flush=True)
    try:
        import flashinfer
        w = flashinfer.prefill.single_prefill_with_kv_cache
        cands.append(("flashinfer single_prefill (auto backend)",
                      lambda: w(q[0], k[0], v[0], causal=False)))
        cands.append(("flashinfer single_prefill (cutlass backend)",
                      lambda: w(q[0], k[0], v[0], causal=False, backend="cutlass")))
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"lib": "flashinfer", "unavailable": repr(e)[:300]}), flush=True)
    cands.append(("torch sdpa (cuDNN / flash backend)",
                  lambda: torch.nn.functional.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2),
                                                                           v.transpose(1, 2))))
    for name, fn in cands:
        try:
            t0 = time.time()
            out = fn()
            if isinstance(out, tuple):
                out = out[0]
            if out.dim() == 3:
                out = out.unsqueeze(0)
            if out.shape[1] == H and out.shape[2] == S:
                out = out.transpose(1, 2)
            err = (out.float() - ref).abs().max().item()
            med, best = timeit(fn)
            print(json.dumps({"lib": name, "ms_median": med, "ms_best": best, "tflops_median": FLOP / med / 1e9,
                              "tflops_best": FLOP / best / 1e9, "max_abs_err_vs_fp32": err,
                              "first_call_s": time.time() - t0}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"lib": name, "failed": repr(e)[:300]}), flush=True)


if __name__ == "__main__":
    main()
