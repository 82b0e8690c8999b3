"""Benchmark: EinSum-graph TFLOP/s of the B200 executor (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config bmm2]
                    [--precision bf16] [--impl ours|reference]

A step is one ed_run of the placed ExecGraph of the config graph (p=8, L=N,
the reference planner's plan from plans/), inputs resident in HBM. `value`
is contraction TFLOP/s = sum over mul/sum join kernels of 2*fp (SURVEY
8(d)) / device time (CUDA events, max over ranks). `e2e` is the same metric
through the C ABI with pinned host buffers: H2D of every input tensor,
on-device chunking, the run, D2H of the assembled output, every step, via
ed_run_steps (the serving loop: step s+1's H2D overlaps step s's compute and
D2H); `e2e.blocking_calls` is the same with one blocking
ed_upload_tensors / ed_run / ed_download sequence per step.
For N > 1 run under torchrun (one process per GPU).
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "EinSum-graph TFLOP/s at 1/2/4/8 B200 and % of tensor peak vs CPU ref"
CONFIG_DESC = {
    "bmm2": "C2 batched contraction bij,bjk->bik b=64, 2048^2, two chained nodes (configs[1])",
    "chain3": "C1 matmul chain ij,jk->ik x3 at 4096^2 (configs[0])",
    "ffnn_big": "C3 FFNN batch 16384 hidden 8192, relu + row softmax (configs[2])",
    "attn_big": "C4 attention s=4096 a=4096 h=32 d=128 (configs[3])",
    "hoc": "C5 abcd,cdef->abef 128^4 (configs[4])",
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["bf16_tflops"], d.get("bf16_tflops_sustained"), d["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.samples.append((time.time(), parts))

    def mark(self, begin):
        if begin:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        # samples that arrived while the timed region ran (nvidia-smi output
        # lags by up to one period, so allow 50 ms of slack)
        t0, t1 = getattr(self, "t0", 0.0), getattr(self, "t1", 1e18)
        inside = [s for t, s in self.samples if t0 <= t <= t1 + 0.05]
        window = "timed region"
        if not inside:  # a region shorter than the sampling period: take the samples right around it
            inside = [s for t, s in self.samples if t0 - 0.15 <= t <= t1 + 0.15]
            window = "timed region +-150 ms"
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[1]) for s in inside if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in inside if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in inside for i in range(4) if s[5 + i].lower().startswith("active")})
        pw = [float(s[3]) for s in inside if s[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside), "power_w_max": max(pw) if pw else None,
                "window": window}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def synthetic_inputs(plan, seed, dtype=np.float32):
    """Synthetic data of the config's shape and distribution: integers in
    [-4,4] for sum/mul-only graphs, U[-1,1) otherwise (runtime.cc:552-571)."""
    rng = np.random.default_rng(seed)
    out = {}
    for vid in plan.input_vertices():
        shape = plan.vertices[vid].bound
        if plan.integer_valued():
            a = rng.integers(-4, 5, size=shape, dtype=np.int8).astype(dtype)
        else:
            a = rng.random(size=shape, dtype=np.float32).astype(dtype) * 2 - 1
        out[vid] = a
    return out


def cpu_baseline(config, threads=True):
    """The reference CPU executor (oracle/_ref, unmodified sources, -O3) on the
    reduced twin of the config: TFLOP/s of execute() alone, threaded with L=8."""
    from oracle import bridge as B
    from paper_2410_02682_b200.plan import Plan
    twin = config.replace("_big", "") + "_s"
    if config == "ffnn_big":
        twin = "ffnn_s"
    if config == "attn_big":
        twin = "attn_s"
    name = f"{twin}_p8_L8"
    doc = json.load(open(os.path.join(ROOT, "plans", name + ".json")))
    plan = Plan.from_json(doc)
    ins = B.generate_inputs(plan, 1)
    kind = "reference" if B.have_ref() else "port"
    if kind == "reference":
        _, secs, _, _ = B.ref_execute(doc, ins, threaded=threads)
    else:
        t0 = time.perf_counter()
        B.oracle_execute(plan, ins)
        secs = time.perf_counter() - t0
    flops = plan.contraction_flops()
    return {"value": flops / secs / 1e12, "unit": "TFLOP/s", "cores": os.cpu_count() if threads else 1,
            "kind": kind, "sample": f"{twin} (reduced twin, SURVEY App. B) p=8 L=8, execute() threaded,"
                                    f" {flops:.3e} contraction flops in {secs:.2f} s",
            "seconds": secs}


def run_reference(args, rank, world):
    if rank != 0:
        return
    vals = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(args.config)
        if i >= args.warmup:
            vals.append(cb["value"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["seconds"] * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generate_inputs)",
            "config": {"workload": CONFIG_DESC.get(args.config, args.config), "graph": args.config,
                       "p": 8, "sample": cb["sample"]},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="bmm2")
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--impl", default="ours")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", default="peer", choices=["nccl", "peer"],
                    help="N > 1: remote chunks read from the producer's HBM over NVLink (CUDA IPC; the "
                         "transport the multi-rank GPU tests run), or NCCL send/recv")
    ap.add_argument("--placement", default="gpu", choices=["gpu", "ref"],
                    help="gpu: GPU-aware re-placement of memory-bound vertices (ed_gpu_placement); "
                         "ref: the reference planner's machine_of")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if os.environ.get("ED_SAME_DEVICE"):  # functional check of N ranks on one GPU (peer transport only)
        local = 0
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    from paper_2410_02682_b200 import build as b
    b.build()
    from paper_2410_02682_b200.executor import Context, PreparedPlan
    from paper_2410_02682_b200.plan import Plan

    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
        idt = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            idt = torch.tensor(list(Context.nccl_unique_id()), dtype=torch.uint8)
        dist.broadcast(idt, 0)
        ctx = Context(local, rank, world, bytes(idt.tolist()) if args.transport == "nccl" else None)
    else:
        ctx = Context(local)

    L = world
    plan = Plan.load(os.path.join(ROOT, "plans", f"{args.config}_p8_L{L}.json"))
    est = None
    if args.placement == "gpu" and L > 1:
        from paper_2410_02682_b200.executor import gpu_placement
        plan, b_ms, a_ms = gpu_placement(plan)
        est = {"est_busiest_ms_ref": b_ms, "est_busiest_ms_gpu": a_ms}
    ins = synthetic_inputs(plan, 1234)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def prepared(**kw):
        pp = PreparedPlan(ctx, plan, precision=args.precision, transport=args.transport, **kw)
        if world > 1 and args.transport == "peer":
            blobs = [None] * world
            torch.distributed.all_gather_object(blobs, pp.peer_export())
            pp.peer_import(blobs)
        return pp

    # ---- device-resident throughput --------------------------------------
    pp = prepared()
    pp.upload(ins)
    with Clocks(local) as clk:
        time.sleep(0.5)  # let the sampler start before the timed region
        for _ in range(args.warmup):
            rep = pp.run()
        barrier()
        torch.cuda.synchronize()
        dev_ms = []
        clk.mark(True)
        for _ in range(args.steps):
            rep = pp.run()
            dev_ms.append(rep.device_ms)
        torch.cuda.synchronize()
        clk.mark(False)
        barrier()
    tot_ms = sum(dev_ms)
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_ms = float(t.item())
    flops = plan.contraction_flops()
    value = flops * args.steps / (tot_ms / 1e3) / 1e12
    launches = rep.gpu_launches
    # chunk bytes this rank sent to peers per step (NCCL or peer transport)
    sent = rep.peer_bytes
    if world > 1:
        t = torch.tensor([float(sent)], dtype=torch.float64)
        torch.distributed.all_reduce(t)
        sent = float(t.item())
    transfers = {"bytes_per_step": sent, "gbs": sent / (tot_ms / args.steps / 1e3) / 1e9 if tot_ms else 0.0,
                 "note": "all ranks' peer bytes / step time (one step moves them concurrently)"}
    pp.close()

    # ---- kernel shares / roofline (one profiled run) -----------------------
    pk, pk_sus, hbm, peak_src = peaks()
    pp = prepared(profile=True)
    pp.upload(ins)
    pp.run()
    pp.run()
    stats = pp.kernel_stats()
    pp.close()
    gemm = [s for s in stats if s["name"].startswith("gemm")]
    g_ms = sum(s["ms"] for s in gemm)
    g_fl = sum(s["flops"] for s in gemm)
    g_n = sum(s["launches"] for s in gemm)
    step_ms = sum(s["ms"] for s in stats)
    traffic = None
    tensor_active = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json"))).get(args.config, {})
        traffic = prof.get("dram_bytes_per_launch")
        tensor_active = [l.get("tensor_active") for l in prof.get("launches", [])] or None
    except Exception:
        pass
    # memory-bound launch classes: achieved algorithmic HBM GB/s against the
    # measured copy bandwidth (the north star's shuffle / elementwise figure)
    for st in stats:
        if st["ms"] > 0 and not st["name"].startswith(("gemm", "attention")):
            st["hbm_gbs"] = st["bytes"] / (st["ms"] / 1e3) / 1e9
            st["hbm_frac"] = st["hbm_gbs"] / hbm
    achieved = g_fl / (g_ms / 1e3) / 1e12 if g_ms else 0.0
    roofline = {"bound": "tensor", "achieved": achieved, "peak": pk, "unit": "TFLOP/s",
                "frac": achieved / pk if pk else None, "traffic": traffic,
                "ncu_tensor_pipe_active": tensor_active,
                "kernel": "tcgen05 GEMM (gemm_kernel)", "launches_per_step": g_n,
                "share_of_step": g_ms / step_ms if step_ms else None,
                "per_launch_tflop": g_fl / max(1, g_n) / 1e12, "peak_source": f"{peak_src} bf16 burst",
                "kernels": stats}

    # ---- end to end through the C ABI ------------------------------------------
    pin = {vid: torch.from_numpy(a).pin_memory() for vid, a in ins.items()}
    pins = {vid: t.numpy() for vid, t in pin.items()}
    outs = {vid: torch.empty(plan.vertices[vid].bound, dtype=torch.float32).pin_memory() for vid in plan.outputs}
    outs_np = {vid: t.numpy() for vid, t in outs.items()}
    pp = prepared()
    h2d = sum(a.nbytes for a in pins.values())
    d2h = sum(a.nbytes for a in outs_np.values())
    pp.upload(pins)
    pp.run()
    pp.download(into=outs_np)
    # (a) blocking calls per step: ed_upload_tensors, ed_run, ed_download
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        pp.upload(pins)
        pp.run()
        pp.download(into=outs_np)
    seq_s = time.perf_counter() - t0
    # (b) the serving loop in one call, ed_run_steps: step s+1's H2D overlaps
    # step s's compute and D2H (copy streams, double-buffered staging)
    pp.run_steps([pins] * 2, [outs_np] * 2)
    barrier()
    t0 = time.perf_counter()
    pp.run_steps([pins] * args.e2e_steps, [outs_np] * args.e2e_steps)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s, seq_s], dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s, seq_s = float(t[0].item()), float(t[1].item())
    pp.close()
    e2e = {"value": flops * args.e2e_steps / e2e_s / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s / args.e2e_steps * 1e3, "api": "ed_run_steps",
           "blocking_calls": {"value": flops * args.e2e_steps / seq_s / 1e12,
                              "ms_per_step": seq_s / args.e2e_steps * 1e3,
                              "api": "ed_upload_tensors + ed_run + ed_download per step"}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(args.config)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": args.precision,
                "data": ("synthetic, numpy-seeded: " + ("integers in [-4,4]" if plan.integer_valued() else "U[-1,1)")
                         + " like generate_inputs (runtime.cc:552-571)"),
                "config": {"workload": CONFIG_DESC.get(args.config, args.config), "graph": args.config,
                           "p": 8, "L": L, "plan": f"plans/{args.config}_p8_L{L}.json",
                           "placement": args.placement if L > 1 else "single GPU", "placement_estimate": est,
                           "transport": args.transport if L > 1 else None,
                           "l2": "inputs larger than L2 (1 GiB per input tensor); no flush needed",
                           "frac_of_peak": value / (pk * world)},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches * args.steps, "clocks": clk.summary(), "transfers": transfers}
        print(json.dumps(line), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
