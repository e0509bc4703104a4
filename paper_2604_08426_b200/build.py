"""Build libkvb.so in-tree for sm_100a (nvcc; static cudart).

``python -m paper_2604_08426_b200.build`` or ``__graft_entry__.build()``.
Objects go to paper_2604_08426_b200/_build/, the library to
paper_2604_08426_b200/libkvb.so (git-ignored, shipped to the GPU box by
gpurun with the snapshot).
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# Experiment builds (A/B runs in one GPU session): KVB_LIB_TAG=<tag> with
# KVB_DEFS="-DNAME=VALUE ..." writes libkvb_<tag>.so from _build_<tag>/; the
# product library is the untagged libkvb.so.
TAG = os.environ.get("KVB_LIB_TAG", "")
DEFS = os.environ.get("KVB_DEFS", "").split() if TAG else []
OBJ = os.path.join(PKG, f"_build_{TAG}" if TAG else "_build")
LIB = os.path.join(PKG, f"libkvb_{TAG}.so" if TAG else "libkvb.so")
SOURCES = ["kvb_api.cu", "kvb_score.cu", "kvb_select.cu", "kvb_attend.cu", "kvb_build.cu",
           "kvb_higgs_tc.cu", "kvb_attend_wh.cu", "kvb_attend_bulk.cu", "kvb_recon.cu", "kvb_tier.cu"]
HEADERS = ["kvb_common.cuh", "kvb_internal.h", "kvb_fuse.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-diag-suppress", "177"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def _digest(paths, extra: str = "") -> str:
    h = hashlib.sha256(extra.encode())
    for p in paths:
        h.update(p.encode())
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def _deps():
    paths = [os.path.join(CSRC, h) for h in HEADERS if os.path.exists(os.path.join(CSRC, h))]
    paths.append(os.path.join(ROOT, "include", "kvb.h"))
    return paths


def _fresh(target: str, digest: str) -> bool:
    stamp = target + ".sha256"
    if not (os.path.exists(target) and os.path.exists(stamp)):
        return False
    with open(stamp) as f:
        return f.read().strip() == digest


def _stamp(target: str, digest: str) -> None:
    with open(target + ".sha256", "w") as f:
        f.write(digest + "\n")


def _compile(src: str, force: bool) -> tuple[str, str, str]:
    """Recompile when the content hash of the source, the shared headers and
    the flags changed (not on mtimes: a shipped object newer than an edited
    source must not be reused)."""
    s = os.path.join(CSRC, src)
    o = os.path.join(OBJ, src.replace(".cu", ".o"))
    cmd = [_nvcc(), *ARCH, *FLAGS, *DEFS, "-c", s, "-o", o]
    digest = _digest([s, *_deps()], " ".join(cmd[1:]))
    if not force and _fresh(o, digest):
        return o, "", digest
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    _stamp(o, digest)
    return o, r.stderr, digest


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, force), srcs))
    objs = [o for o, _, _ in results]
    if verbose:
        for _, log, _ in results:
            if log:
                sys.stderr.write(log)
    lib_digest = hashlib.sha256("".join(d for _, _, d in results).encode()).hexdigest()
    if force or not _fresh(LIB, lib_digest):
        cmd = [_nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-Xcompiler", "-fPIC"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        _stamp(LIB, lib_digest)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
