"""Builds libed_gpu.so in-tree (nvcc, sm_100a only).

    python -m paper_2410_02682_b200.build
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libed_gpu.so")
SOURCES = ["api.cu", "plan.cu", "build.cu", "alloc.cu", "exec.cu", "io.cu", "placement.cu", "gemm_sm100.cu",
           "kernels.cu", "ewise.cu", "attn_sm100.cu", "attn_x3_sm100.cu"]
HEADERS = ["runtime.h", "libm_exp.cuh", "ptx.cuh", "gemm_sm100.h", "kernels.h", "ewise.h", "attn_sm100.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# The toolchain's libstdc++.so link is missing (only the .a resolves); a static
# libstdc++ inside a dlopen'ed .so clashes with the host's, so link the system
# shared one explicitly.
STDCXX = "/usr/lib/x86_64-linux-gnu/libstdc++.so.6"


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "ed_gpu.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    common = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
              "-I" + os.path.join(ROOT, "include"), "-I" + CSRC] + ARCH
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [_nvcc()] + common + ["-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + out.decode())
    link = [_nvcc(), "-shared"] + ARCH + objs + ["-o", LIB + ".tmp", "-lcudart", "-lnccl", "-Xlinker", STDCXX]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + " ".join(link) + "\n" + r.stdout.decode())
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
