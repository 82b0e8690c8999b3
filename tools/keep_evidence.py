"""Copy one gpurun evidence pass (tools/gpu_final_*.sh) into tracked summaries
under profiles/.

    python tools/keep_evidence.py <gpurun_out/subdir> <tag>

Writes profiles/<tag>_bench_all.jsonl (every bench line of the pass, the
default headline first, then the reference arm), <tag>_launches.md (the ncu
launch list of the default bench command, per kernel), <tag>_ncu_full.md
(the `ncu --set full` capture of the headline kernel, tracked metrics),
<tag>_pytest_gpu.txt (the GPU suite's tail) and refreshes
profiles/r02_traffic.json (the kept DRAM traffic bench.py reports).
"""
import glob
import json
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_profiles import launches  # noqa: E402
from ncu_summary import main as ncu_rows  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last_json(path):
    lines = [ln for ln in open(path).read().splitlines() if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def main(src, tag):
    out = os.path.join(ROOT, "profiles")
    lines = []
    for name in ["bench_default.jsonl", "bench_reference.jsonl"] + sorted(
            os.path.basename(p) for p in glob.glob(os.path.join(src, "bench_*_*.jsonl"))):
        p = os.path.join(src, name)
        if name in ("bench_default.jsonl", "bench_reference.jsonl") and lines and any(
                ln.get("_file") == name for ln in lines):
            continue
        if os.path.exists(p):
            d = last_json(p)
            if d is not None:
                d["_file"] = name
                lines.append(d)
    with open(os.path.join(out, f"{tag}_bench_all.jsonl"), "w") as f:
        for d in lines:
            f.write(json.dumps(d) + "\n")
    lp = os.path.join(src, "launches_default.csv")
    if os.path.exists(lp):
        L = launches(lp)
        tot = sum(v[1] for v in L.values())
        with open(os.path.join(out, f"{tag}_launches.md"), "w") as f:
            f.write(f"# {tag}: ncu launch list of the default bench command\n\n")
            f.write("`ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 1 "
                    "--extras '' --no-cpu-baseline --e2e-steps 1` (cold-cache, serialised: compare shares, not "
                    "absolutes). Includes the device input generation, chunking and the e2e leg's launches.\n\n")
            f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
            for k, (n, ns) in sorted(L.items(), key=lambda kv: -kv[1][1]):
                f.write(f"| `{k}` | {n} | {ns / 1e6:.3f} | {ns / tot:.1%} |\n")
    reps = glob.glob(os.path.join(src, "*.ncu-rep"))
    if reps:
        with open(os.path.join(out, f"{tag}_ncu_full.md"), "w") as f:
            for rp in sorted(reps):
                f.write(f"# {tag}: `ncu --set full --clock-control none --import-source on` ({os.path.basename(rp)})\n\n")
                for i, d in enumerate(ncu_rows(rp)):
                    f.write(f"## launch {i}\n\n| metric | value |\n|---|---|\n")
                    for k, v in d.items():
                        f.write(f"| `{k}` | {v} |\n")
                    f.write("\n")
    tp = os.path.join(src, "r02_traffic.json")
    if os.path.exists(tp):
        shutil.copy(tp, os.path.join(out, "r02_traffic.json"))
    pp = os.path.join(src, "pytest_gpu.log")
    if os.path.exists(pp):
        tail = open(pp).read().splitlines()[-12:]
        with open(os.path.join(out, f"{tag}_pytest_gpu.txt"), "w") as f:
            f.write("\n".join(tail) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
