"""Build the in-tree sm_100a library ``libff_chain.so`` with nvcc.

    python -m paper_2512_12949_b200.build
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libff_chain.so")
SOURCES = ("ff_chain.cu", "dsm_primitives.cu")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    built = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "ff_chain.h"))
    return any(os.path.getmtime(p) > built for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    """defines: extra -D flags for A/B builds of kernel variants (written to another `out`)."""
    if not force and out == OUT and not _stale():
        return OUT
    cmd = [nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-cudart", "static", *[f"-D{d}" for d in defines], "-o", out + ".tmp"]
    cmd += [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    # python -m paper_2512_12949_b200.build [--force] [-v] [-DNAME=VAL ... --out path.so]
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else OUT
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=out, defines=defs))
