"""DRAM traffic per launch of each config's dominant kernel (ncu), tied to the
exact library sources it was measured on (bench.py's csrc_sha), so bench.py
can report roofline.traffic without ever quoting a stale capture.

    python tools/capture_traffic.py OUT.json hoc:fp32x3 hoc:bf16 bmm2_repart:fp32x3 ...

Runs on the GPU box: one `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum --clock-control none` capture of tools/kernel_times.py per
config, keeping the contraction kernels' launches (one profiled run).
"""
import csv
import io
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def capture(config, prec):
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:gemm_|attn_", "--csv",
           sys.executable, os.path.join(ROOT, "tools", "kernel_times.py"), f"{config}_p8_L1", "1", prec]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900).stdout
    rows = list(csv.reader(io.StringIO("\n".join(l for l in out.splitlines() if l.startswith('"')))))
    if not rows:
        return None
    h = rows[0]
    per = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        per.setdefault(d["ID"], {"kernel": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"])
    # kernel_times.py warms up 3 runs, then one timed run: the last run's launches
    launches = list(per.values())
    n_per_run = len(launches) // 4 if len(launches) % 4 == 0 else len(launches)
    last = launches[-n_per_run:]
    byts = [l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"] for l in last]
    return {"dram_bytes_per_launch": sum(byts) / len(byts), "launches": last,
            "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none on "
                      f"tools/kernel_times.py {config}_p8_L1 1 {prec} ({time.strftime('%Y-%m-%d')})"}


def main():
    from bench import csrc_sha
    out_path = sys.argv[1]
    doc = {"entries": {}}
    if os.path.exists(out_path):
        doc = json.load(open(out_path))
    sha = csrc_sha()
    for spec in sys.argv[2:]:
        config, prec = spec.split(":")
        e = capture(config, prec)
        if e:
            e["csrc_sha"] = sha
            doc["entries"][f"{config}/{prec}"] = e
            print(spec, e["dram_bytes_per_launch"])
    with open(out_path, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
