"""Benchmark: EinSum-graph TFLOP/s of the B200 executor (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config hoc]
                    [--precision fp32x3] [--impl ours|reference]

A step is one ed_run of the placed ExecGraph of the config graph (p=8, L=N,
the reference planner's plan from plans/), inputs resident in HBM. The
default workload is the largest config, C5 hoc (abcd,cdef->abef at 128^4,
8.8 TFLOP per step), in the fp32-accurate mode (fp32x3: three TF32 tensor
products hi*hi + hi*lo + lo*hi per contraction, fp32 storage — the class of
the reference's f32 mode, runtime.h:39-43), so `dtype` is no narrower than
the reference's f32 arithmetic. `value` is contraction TFLOP/s = sum over
mul/sum joins of 2*fp / device time (CUDA events, max over
ranks). The same line carries the bf16 tensor-core mode of the same config
(`bf16`) and C2's repartition variant (`bmm2_repart`, batch-sharded Z1 into
row-sharded Z2) in both modes, each with its own roofline. Inputs are the
reference's generate_inputs stream (runtime.cc:552-571), drawn on the device
by ed_generate_inputs bit for bit. `e2e` is the same metric through the C ABI
with pinned host buffers: H2D of every input tensor, on-device chunking, the
run, D2H of the assembled output, every step, via ed_run_steps.
For N > 1 run under torchrun (one process per GPU).
"""
import argparse
import ctypes as C
import hashlib
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
    "bmm2": "C2 batched contraction bij,bjk->bik b=64, 2048^2, two chained nodes (configs[1]), DP plan",
    "bmm2_repart": "C2 batched contraction bij,bjk->bik b=64, 2048^2 with repartition between nodes (configs[1]): "
                   "Z1 batch-sharded d=[8,1,1,8,1,1], Z2 row-sharded d=[1,8,1,1,1,1]",
    "chain3": "C1 matmul chain ij,jk->ik x3 at 4096^2 (configs[0])",
    "ffnn_big": "C3 FFNN batch 16384 hidden 8192, relu + row softmax (configs[2])",
    "attn_big": "C4 attention s=4096 a=4096 h=32 d=128 (configs[3])",
    "hoc": "C5 higher-order contraction abcd,cdef->abef 128^4 (configs[4], the largest config)",
}
# reduced / mid-scale twins the CPU reference runs on (full size is hours on the host)
CPU_TWIN = {"hoc": "hoc_m", "bmm2": "bmm2_s", "bmm2_repart": "bmm2_s_repart", "chain3": "chain3_s",
            "ffnn_big": "ffnn_s", "attn_big": "attn_s"}
TF32_NOMINAL = 1100.0  # dense TF32 TFLOP/s per B200 (B200_PROFILING.md nominal table)


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


def csrc_sha():
    """sha256 over the library's sources: ties a kept ncu traffic figure to the
    code it was measured on (profiles/r02_traffic.json)."""
    from paper_2410_02682_b200 import build as b
    h = hashlib.sha256()
    for f in b.SOURCES + b.HEADERS:
        with open(os.path.join(b.CSRC, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def kept_traffic(config, precision, sha):
    """DRAM bytes per launch of the config's dominant kernel from the ncu
    capture of the same command (tools/capture_traffic.py), only if it was
    taken on these exact sources; otherwise None (never a stale figure)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            e = json.load(f)["entries"][f"{config}/{precision}"]
    except Exception:
        return None, "no ncu capture kept for this config/precision"
    if e.get("csrc_sha") != sha:
        return None, f"kept capture is of other sources ({e.get('csrc_sha')}); not reported"
    return e["dram_bytes_per_launch"], e.get("source")


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(config, runs=3):
    """The reference CPU executor (oracle/_ref: the unmodified reference
    sources, g++ -O3) timed on the host: execute() alone, threaded mode
    (runtime.cc:301-355, one worker thread per machine, L = 8) on the
    config's CPU-sized twin, median of `runs`. Falls back to the oracle's
    single-threaded restatement if the reference build is absent."""
    from oracle import bridge as B
    from paper_2410_02682_b200.plan import Plan
    twin = CPU_TWIN.get(config, config + "_s")
    name = f"{twin}_p8_L8"
    doc = json.load(open(os.path.join(ROOT, "plans", name + ".json")))
    plan = Plan.from_json(doc)
    ins = B.generate_inputs(plan, 1)
    kind = "reference" if B.have_ref() else "port"
    secs = []
    for _ in range(runs):
        if kind == "reference":
            secs.append(B.ref_execute(doc, ins, threaded=True)[1])
        else:
            t0 = time.perf_counter()
            B.oracle_execute(plan, ins)
            secs.append(time.perf_counter() - t0)
    sec = statistics.median(secs)
    flops = plan.contraction_flops()
    threads = plan.n_machines if kind == "reference" else 1
    return {"value": flops / sec / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": kind,
            "sample": f"{twin} (CPU-sized twin of {config}; graphs/{twin}.eg) p=8 L={plan.n_machines}, reference "
                      f"execute() in threaded mode with {threads} worker threads, f64, {flops:.3e} contraction "
                      f"flops, median of {runs} runs = {sec:.2f} s",
            "cpu_model": cpu_model(), "host_threads_available": os.cpu_count(), "seconds": sec,
            "runs_s": secs}


def run_reference(args, rank, world):
    """--impl reference: the reference's own executor on the host cores, one
    bounded sample of the workload (its CPU twin) per step; rank 0 only."""
    if rank != 0:
        return
    vals, cb = [], None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(args.config, runs=1)
        if i >= args.warmup:
            vals.append(cb["value"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["seconds"] * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generate_inputs, runtime.cc:552-571)",
            "config": {"workload": CONFIG_DESC.get(args.config, args.config), "graph": args.config, "p": 8,
                       "sample": cb["sample"]},
            "cpu_baseline": {"value": v, **{k: cb[k] for k in ("unit", "cores", "kind", "sample", "cpu_model")},
                             "statistic": f"median of {args.steps} steps"},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def roofline_of(stats, precision, pk, pk_sus, hbm, peak_src, traffic=None, traffic_note=None, tf32_meas=None):
    """Roofline of the dominant kernel class (the tcgen05 contractions) from a
    profiled run's per-launch event times: achieved = algorithmic contraction
    flops per launch / mean launch time."""
    gemm = [s for s in stats if s["name"].startswith(("gemm", "attention"))]
    g_ms = sum(s["ms"] for s in gemm)
    g_fl = sum(s["flops"] for s in gemm)
    g_n = sum(s["launches"] for s in gemm)
    step_ms = sum(s["ms"] for s in stats)
    for st in stats:  # memory-bound launch classes: algorithmic GB/s vs the measured copy bandwidth
        if st["ms"] > 0 and not st["name"].startswith(("gemm", "attention")):
            st["hbm_gbs"] = st["bytes"] / (st["ms"] / 1e3) / 1e9
            st["hbm_frac"] = st["hbm_gbs"] / hbm
    achieved = g_fl / (g_ms / 1e3) / 1e12 if g_ms else 0.0
    if precision == "fp32x3":
        peak = TF32_NOMINAL / 3
        src = ("nominal dense TF32 (1100 TFLOP/s, B200_PROFILING.md) / 3: the kernel runs three TF32 products per "
               "algorithmic flop; MEASURED_PEAKS.json has no TF32 figure")
        alt = {"tensor_tf32_products_tflops": achieved * 3}
        if tf32_meas:
            alt["frac_of_measured_cublas_tf32_div3"] = achieved / (tf32_meas / 3)
            alt["measured_cublas_tf32_tflops"] = tf32_meas
        alt["frac_of_measured_bf16_div6"] = achieved / (pk / 6)
    elif precision == "tf32":
        peak, src, alt = TF32_NOMINAL, "nominal dense TF32 (B200_PROFILING.md)", {}
    else:
        peak, src, alt = pk, f"{peak_src} bf16 burst (MEASURED_PEAKS.json)", {
            "frac_of_sustained": achieved / pk_sus if pk_sus else None}
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None, "traffic": traffic, "traffic_source": traffic_note,
            "kernel": "tcgen05 contraction (gemm_kernel / attn_kernel)", "launches_per_step": g_n,
            "share_of_step": g_ms / step_ms if step_ms else None, "per_launch_tflop": g_fl / max(1, g_n) / 1e12,
            "peak_source": src, "alternatives": alt, "kernels": stats}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="hoc")
    ap.add_argument("--precision", default="fp32x3")
    ap.add_argument("--impl", default="ours")
    # e2e steps: the serving loop's steady state (12 steps: 56 ms/step on hoc, the copy
    # pipeline's fill and drain not yet amortised; 32: 53.5 ms)
    ap.add_argument("--e2e-steps", type=int, default=32)
    ap.add_argument("--extras", default="bf16,bmm2_repart",
                    help="comma list of extra measurements in the same line: bf16 (this config in bf16), "
                         "bmm2_repart (C2's repartition variant, fp32x3 and bf16); '' for none")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", default="peer", choices=["nccl", "peer"],
                    help="N > 1: remote chunks read from the producer's HBM over NVLink (CUDA IPC; the "
                         "transport the multi-rank GPU tests run), or NCCL send/recv (opt-in, unverified)")
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
        nid = None
        if args.transport == "nccl":
            idt = torch.zeros(128, dtype=torch.uint8)
            if rank == 0:
                idt = torch.tensor(list(Context.nccl_unique_id()), dtype=torch.uint8)
            dist.broadcast(idt, 0)
            nid = bytes(idt.tolist())
        ctx = Context(local, rank, world, nid)
    else:
        ctx = Context(local)

    L = world

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(*xs):
        if world == 1:
            return xs
        t = torch.tensor(list(xs), dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return tuple(float(v) for v in t.tolist())

    def load_plan(config):
        plan = Plan.load(os.path.join(ROOT, "plans", f"{config}_p8_L{L}.json"))
        est = None
        if args.placement == "gpu" and L > 1:
            from paper_2410_02682_b200.executor import gpu_placement
            plan, b_ms, a_ms = gpu_placement(plan)
            est = {"est_busiest_ms_ref": b_ms, "est_busiest_ms_gpu": a_ms}
        return plan, est

    def prepared(plan, precision, **kw):
        pp = PreparedPlan(ctx, plan, precision=precision, transport=args.transport, **kw)
        if world > 1 and args.transport == "peer":
            blobs = [None] * world
            torch.distributed.all_gather_object(blobs, pp.peer_export())
            pp.peer_import(blobs)
        return pp

    pk, pk_sus, hbm, peak_src = peaks()
    tf32_meas = None
    try:
        tf32_meas = json.load(open(os.path.join(ROOT, "profiles", "r02_tf32_peak.json")))["tf32_tflops"]
    except Exception:
        pass
    sha = csrc_sha()

    def measure(config, precision, steps, clk=None):
        """Device-resident throughput of one config/precision, then one
        profiled run for the per-kernel roofline. Returns (summary, plan, est)."""
        plan, est = load_plan(config)
        pp = prepared(plan, precision)
        pp.generate_inputs(1)
        for _ in range(args.warmup):
            rep = pp.run()
        barrier()
        torch.cuda.synchronize()
        dev_ms = []
        if clk:
            clk.mark(True)
        for _ in range(steps):
            rep = pp.run()
            dev_ms.append(rep.device_ms)
        torch.cuda.synchronize()
        if clk:
            clk.mark(False)
        barrier()
        (tot_ms,) = max_over_ranks(sum(dev_ms))
        sent = float(rep.peer_bytes)
        if world > 1:
            t = torch.tensor([sent], dtype=torch.float64)
            torch.distributed.all_reduce(t)
            sent = float(t.item())
        launches = rep.gpu_launches
        barrier()
        pp.close()
        flops = plan.contraction_flops()
        pp = prepared(plan, precision, profile=True)
        pp.generate_inputs(1)
        pp.run()
        pp.run()
        stats = pp.kernel_stats()
        barrier()
        pp.close()
        traffic, tsrc = kept_traffic(config, precision, sha)
        value = flops * steps / (tot_ms / 1e3) / 1e12
        return {"value": value, "unit": "TFLOP/s", "ms_per_step": tot_ms / steps, "steps": steps,
                "dtype": precision, "flops_per_step": flops, "launches_per_step": launches,
                "roofline": roofline_of(stats, precision, pk, pk_sus, hbm, peak_src, traffic, tsrc, tf32_meas),
                "transfers": {"bytes_per_step": sent, "gbs": sent / (tot_ms / steps / 1e3) / 1e9 if tot_ms else 0.0,
                              "note": "all ranks' peer bytes / step time"}}, plan, est

    # ---- headline: device-resident throughput ----------------------------------
    with Clocks(local) as clk:
        time.sleep(0.5)  # let the sampler start before the timed region
        head, plan, est = measure(args.config, args.precision, args.steps, clk)
    clocks = clk.summary()

    extras = {}
    want = [e for e in args.extras.split(",") if e]
    if "bf16" in want and args.precision != "bf16":
        extras["bf16"], _, _ = measure(args.config, "bf16", args.steps)
    if "bmm2_repart" in want and args.config != "bmm2_repart":
        extras["bmm2_repart"] = {"workload": CONFIG_DESC["bmm2_repart"]}
        for prec in (args.precision, "bf16"):
            extras["bmm2_repart"][prec], _, _ = measure("bmm2_repart", prec, args.steps)

    # ---- end to end through the C ABI -------------------------------------------
    # host inputs: the same generate_inputs stream, read back once into pinned memory
    pp = prepared(plan, args.precision)
    pp.generate_inputs(1)
    ins = {vid: torch.empty(plan.vertices[vid].bound, dtype=torch.float32).pin_memory()
           for vid in plan.input_vertices()}
    pins = {vid: t.numpy() for vid, t in ins.items()}
    pp.download(into=pins, vertices=list(pins))
    outs = {vid: torch.empty(plan.vertices[vid].bound, dtype=torch.float32).pin_memory() for vid in plan.outputs}
    outs_np = {vid: t.numpy() for vid, t in outs.items()}
    h2d = sum(a.nbytes for a in pins.values())
    d2h = sum(a.nbytes for a in outs_np.values())
    pp.upload(pins)
    pp.run()
    pp.download(into=outs_np)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        pp.upload(pins)
        pp.run()
        pp.download(into=outs_np)
    seq_s = time.perf_counter() - t0
    pp.run_steps([pins] * 2, [outs_np] * 2)
    barrier()
    t0 = time.perf_counter()
    pp.run_steps([pins] * args.e2e_steps, [outs_np] * args.e2e_steps)
    e2e_s = time.perf_counter() - t0
    e2e_s, seq_s = max_over_ranks(e2e_s, seq_s)
    barrier()  # no rank frees IPC-exported memory while a peer may still read it
    pp.close()
    flops = plan.contraction_flops()
    e2e = {"value": flops * args.e2e_steps / e2e_s / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s / args.e2e_steps * 1e3, "api": "ed_run_steps",
           "blocking_calls": {"value": flops * args.e2e_steps / seq_s / 1e12,
                              "ms_per_step": seq_s / args.e2e_steps * 1e3,
                              "api": "ed_upload_tensors + ed_run + ed_download per step"}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(args.config)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "host_threads_available")}

    if rank == 0:
        roof = head.pop("roofline")
        line = {"metric": METRIC, "value": head["value"], "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": args.precision,
                "data": ("synthetic: the reference's generate_inputs stream (runtime.cc:552-571, std::mt19937_64, "
                         + ("integers in [-4,4]" if plan.integer_valued() else "U[-1,1)")
                         + ") drawn on the device by ed_generate_inputs, bit-exact with libstdc++"),
                "config": {"workload": CONFIG_DESC.get(args.config, args.config), "graph": args.config,
                           "p": 8, "L": L, "plan": f"plans/{args.config}_p8_L{L}.json",
                           "precision_note": ("fp32x3 = fp32 storage, contractions as three TF32 tensor products "
                                              "hi*hi + hi*lo + lo*hi accumulated in fp32 (the reference's f32 "
                                              "class; bit-exact on this integer graph)") if args.precision == "fp32x3"
                           else None,
                           "placement": args.placement if L > 1 else "single GPU", "placement_estimate": est,
                           "transport": args.transport if L > 1 else None,
                           "l2": "inputs larger than L2 (>= 1 GiB per input tensor); no flush needed",
                           "frac_of_peak": roof["frac"]},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": head["launches_per_step"] * args.steps, "clocks": clocks,
                "transfers": head["transfers"], "csrc_sha": sha, **extras}
        print(json.dumps(line), flush=True)
    barrier()
    ctx.close()


if __name__ == "__main__":
    main()
