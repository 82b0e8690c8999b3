import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PLANS = os.path.join(ROOT, "plans")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libed_gpu.so)")


def load_plan(name):
    from paper_2410_02682_b200.plan import Plan
    return Plan.load(os.path.join(PLANS, name + ".json"))


def load_doc(name):
    with open(os.path.join(PLANS, name + ".json")) as f:
        return json.load(f)


def golden_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(case):
    """-> (plan name, inputs {vid: f64}, out64, out32, counters, total)"""
    z = np.load(os.path.join(GOLDEN, case + ".npz"))
    name = case.rsplit("_s", 1)[0]
    ins = {int(k[3:]): z[k] for k in z.files if k.startswith("in_")}
    o64 = {int(k[6:]): z[k] for k in z.files if k.startswith("out64_")}
    o32 = {int(k[6:]): z[k] for k in z.files if k.startswith("out32_")}
    orc = {int(k[7:]): z[k] for k in z.files if k.startswith("oracle_")}
    return name, ins, o64, o32, orc, [tuple(int(x) for x in r) for r in z["counters"]], int(z["total"])


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu_ctx():
    if not gpu_available():
        pytest.skip("no CUDA device")
    from paper_2410_02682_b200 import build
    build.build()
    from paper_2410_02682_b200.executor import Context
    ctx = Context(0)
    yield ctx
    ctx.close()
