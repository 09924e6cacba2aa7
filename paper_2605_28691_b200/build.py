"""Build libosp_skiparse.so in-tree with nvcc for sm_100a (no torch JIT cache)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = Path(os.environ["OSP_LIB_OUT"]) if os.environ.get("OSP_LIB_OUT") else PKG / "libosp_skiparse.so"
SOURCES = ["abi.cu", "rearrange.cu", "attn_fwd.cu", "attn_bwd.cu", "hif8.cu", "proj.cu", "peer.cu", "debug_mma.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
    deps.append(ROOT / "include" / "osp_skiparse.h")
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    objs = []
    jobs = []
    for s in SOURCES:
        obj = LIB.parent / (LIB.name + "." + s + ".o")
        cmd = [NVCC, "-c", str(CSRC / s), "-o", str(obj), "-O3", "-std=c++17",
               "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
               "-Xcompiler", "-fPIC", "-I", str(ROOT / "include"), "--expt-relaxed-constexpr",
               *os.environ.get("OSP_NVCC_FLAGS", "").split()]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        jobs.append((cmd, s))
        objs.append(str(obj))
    procs = [(subprocess.Popen(c, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True), s)
             for c, s in jobs]
    failed = False
    for p, s in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(f"--- nvcc {s}\n{out}")
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.check_call([NVCC, "-shared", "-o", str(tmp), *objs, "-cudart", "static",
                           "-gencode", "arch=compute_100a,code=sm_100a"])
    os.replace(tmp, LIB)
    for o in objs:
        os.unlink(o)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
