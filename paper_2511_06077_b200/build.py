"""Build libstca.so (the C-ABI library of include/stca.h) in-tree for sm_100a.

    python -m paper_2511_06077_b200.build [--force] [--verbose]

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3; objects are built in
parallel under build/ and linked into paper_2511_06077_b200/libstca.so (git-ignored,
but it travels to the GPU box with the gpurun snapshot).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libstca.so")
BUILD = os.path.join(ROOT, "build", "stca")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["api.cu", "kernels_cc.cu", "tc_gemm.cu", "tc_host.cu", "tc_proj.cu", "tc_attn.cu", "tc_attn_wide.cu", "tc_attn_narrow.cu", "rlb_batch.cu",
           "encode.cu", "tc_attn_pair.cu", "tc_chain.cu",
           "tc_attn_bwd.cu", "hist_bwd.cu", "stack_bwd.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def source_digest() -> str:
    """sha256 over the library's sources, its header and the compile flags: identifies a BUILD by what it
    was built from (nvcc output is not bit-reproducible, so the binary's own hash changes on a rebuild of
    the same sources).  Profiles keyed by it stay valid across rebuilds."""
    import hashlib
    h = hashlib.sha256()
    h.update(" ".join(ARCH + FLAGS[:-1]).encode())
    for name in sorted(os.listdir(CSRC)):
        h.update(name.encode())
        with open(os.path.join(CSRC, name), "rb") as f:
            h.update(f.read())
    with open(os.path.join(ROOT, "include", "stca.h"), "rb") as f:
        h.update(f.read())
    return h.hexdigest()


def _deps_mtime() -> float:
    m = os.path.getmtime(os.path.join(ROOT, "include", "stca.h"))
    for f in os.listdir(CSRC):
        m = max(m, os.path.getmtime(os.path.join(CSRC, f)))
    return m


def _compile(src: str, verbose: bool, defines=(), build_dir: str = BUILD) -> str:
    obj = os.path.join(build_dir, src + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, *["-D" + d for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(build_dir, src + ".log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
    if p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
        raise RuntimeError(f"nvcc failed for {src} (see {log})")
    if verbose:
        sys.stderr.write(p.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, defines=(), variant: str = "") -> str:
    """variant/defines: an A/B build (e.g. -DSTCA_NARROW_PF=0) as libstca_<variant>.so, loaded with
    STCA_LIB=<path>; never used by the product's default import."""
    out = OUT if not variant else os.path.join(PKG, f"libstca_{variant}.so")
    bdir = BUILD if not variant else os.path.join(ROOT, "build", "stca_" + variant)
    if not force and os.path.exists(out) and os.path.getmtime(out) >= _deps_mtime():
        return out
    os.makedirs(bdir, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(SOURCES))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, defines, bdir), SOURCES))
    tmp = out + ".tmp"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-lcublas"])
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--variant", default="")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(a.force, a.verbose, a.defines, a.variant))
