"""Turn gpurun_out/ ncu artefacts into tracked summaries under profiles/.

    python tools/make_profiles.py <round tag> <config>
"""
import csv
import json
import os
import sys
from collections import OrderedDict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import main as ncu_rows  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        ns = float(r[vi].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    return agg


def main(tag, config):
    out = os.path.join(ROOT, "profiles")
    os.makedirs(out, exist_ok=True)
    L = launches(os.path.join(ROOT, "gpurun_out", "launches.csv"))
    tot = sum(v[1] for v in L.values())
    with open(os.path.join(out, f"{tag}_launches_{config}.md"), "w") as f:
        f.write(f"# {tag}: ncu launch list, `bench.py --config {config} --steps 2 --warmup 1`\n\n")
        f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised; "
                "compare shares, not absolutes). Includes upload/chunking and e2e launches of the bench process.\n\n")
        f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, (n, ns) in sorted(L.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| `{k}` | {n} | {ns / 1e6:.3f} | {ns / tot:.1%} |\n")
    rows = ncu_rows(os.path.join(ROOT, "gpurun_out", "gemm_prof.ncu-rep"))
    with open(os.path.join(out, f"{tag}_gemm_ncu_{config}.md"), "w") as f:
        f.write(f"# {tag}: `ncu --set full` of the tcgen05 GEMM ({config})\n\n")
        for i, d in enumerate(rows):
            f.write(f"## launch {i}\n\n| metric | value |\n|---|---|\n")
            for k, v in d.items():
                f.write(f"| `{k}` | {v} |\n")
            f.write("\n")
    traffic = []
    for d in rows:
        rd = float(d["dram__bytes_read.sum"].split()[0]) * (1e9 if "Gbyte" in d["dram__bytes_read.sum"] else 1e6)
        wr = float(d["dram__bytes_write.sum"].split()[0]) * (1e9 if "Gbyte" in d["dram__bytes_write.sum"] else 1e6)
        traffic.append(rd + wr)
    sp = os.path.join(out, "ncu_summary.json")
    summ = json.load(open(sp)) if os.path.exists(sp) else {}
    summ[config] = {"round": tag, "dram_bytes_per_launch": sum(traffic) / len(traffic),
                    "launches": [{"time": d["gpu__time_duration.sum"],
                                  "tensor_active": d.get("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                                  "dram_read": d["dram__bytes_read.sum"], "dram_write": d["dram__bytes_write.sum"]}
                                 for d in rows]}
    json.dump(summ, open(sp, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
