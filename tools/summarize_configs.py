"""profiles/<tag>_configs.md from gpurun_out/prof/ (bench lines + ncu launch lists)."""
import csv, json, os, sys
from collections import OrderedDict
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = os.path.join(ROOT, "gpurun_out", "prof")
out = [f"# {tag}: all configs (bf16 mode, p=8, L=1, one B200)\n",
       "Per-kernel times come from the bench's profiled run (CUDA events around each launch, warm L2 between "
       "launches of a step); DRAM bytes from `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum` over the "
       "same step (cold, serialised launches). `alg GB/s` = algorithmic bytes / event time.\n"]
for c in ["bmm2", "chain3", "hoc", "ffnn_big", "attn_big"]:
    lines = [l for l in open(os.path.join(src, f"bench_{c}.jsonl")).read().splitlines() if l.startswith("{")]
    d = json.loads(lines[-1])
    out.append(f"\n## {c} — {d['value']:.1f} TFLOP/s, {d['ms_per_step']:.3f} ms/step, GEMM roofline frac "
               f"{d['roofline']['frac']:.3f} (of measured {d['roofline']['peak']} TFLOP/s), clocks {d['clocks']}\n")
    out.append("| launch class | launches/step | ms | TFLOP/s | alg GB/s |\n|---|---|---|---|---|")
    for k in d["roofline"]["kernels"]:
        n = k["launches"]
        tf = k["flops"] / (k["ms"] / 1e3) / 1e12 if k["flops"] and k["name"].startswith("gemm") else 0
        gb = k["bytes"] / (k["ms"] / 1e3) / 1e9 if k["ms"] else 0
        out.append(f"| `{k['name']}` | {n:g} | {k["ms"]:.3f} | {tf:.0f} | {gb:.0f} |")
    rows = [r for r in csv.reader(open(os.path.join(src, f"launches_{c}.csv"))) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        a = agg.setdefault(name, {"n": 0, "gpu__time_duration.sum": 0.0, "dram__bytes_read.sum": 0.0,
                                  "dram__bytes_write.sum": 0.0})
        v = float(r[vi].replace(",", ""))
        a[r[mi]] = a.get(r[mi], 0.0) + v
        if r[mi] == "gpu__time_duration.sum":
            a["n"] += 1
    out.append("\nncu launch list (whole bench process: upload, warm-up, profiled and e2e steps):\n")
    out.append("| kernel | launches | total ms | DRAM read GB | DRAM write GB |\n|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        out.append(f"| `{k}` | {a['n']} | {a['gpu__time_duration.sum']/1e6:.3f} | "
                   f"{a['dram__bytes_read.sum']/1e9:.2f} | {a['dram__bytes_write.sum']/1e9:.2f} |")
open(os.path.join(ROOT, "profiles", f"{tag}_configs.md"), "w").write("\n".join(out) + "\n")
