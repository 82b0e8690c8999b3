"""The product path never routes through the oracle, and fails loudly without
its CUDA library (no CPU fallback)."""
import os
import re
import subprocess
import sys

from conftest import ROOT

PKG = os.path.join(ROOT, "paper_2410_02682_b200")


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if not f.endswith((".py", ".cu", ".cuh", ".h", ".cc")):
                continue
            text = open(os.path.join(dirpath, f)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle\b", text, re.M), f
            assert "liboracle" not in text and "oracle/_ref" not in text, f


def test_missing_library_fails_loudly():
    env = dict(os.environ, ED_LIB_PATH=os.path.join(ROOT, "no_such_libed_gpu.so"))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2410_02682_b200.executor import library\n"
            "try:\n    library()\nexcept ImportError as e:\n    print('raised', e)\n" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert "raised" in out.stdout, out.stdout + out.stderr
