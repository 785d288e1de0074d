"""In-tree build of libtilefuse.so (sm_100a) with nvcc.

    python -m paper_2605_02953_b200._build        # or __graft_entry__.build()

The shared library is written next to this file so it travels with the repo
snapshot to the GPU box.  cudart is linked statically and the driver API is
reached through cudaGetDriverEntryPoint, so the library also loads on a host
without a GPU driver (the CPU tests only check its exported symbols).
"""

from __future__ import annotations

import hashlib
import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libtilefuse.so"
SOURCES = ["tf_team.cu", "tf_ops.cu", "tf_gemm.cu", "tf_moe.cu", "tf_attn.cu", "tf_mega.cu", "tf_layer.cu", "tf_prep.cu", "tf_agmoe.cu", "tf_nvls.cu", "tf_topo.cu", "tf_swizzle.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libtilefuse")
    return cand


def _digest() -> str:
    h = hashlib.sha256()
    h.update(os.environ.get("TF_NVCC_EXTRA", "").encode())
    for p in sorted(list(CSRC.glob("*")) + [ROOT / "include" / "tilefuse.h", pathlib.Path(__file__)]):
        if p.is_file():
            h.update(p.name.encode())
            h.update(p.read_bytes())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False) -> pathlib.Path:
    stamp = PKG / ".libtilefuse.stamp"
    digest = _digest()
    if LIB.exists() and stamp.exists() and stamp.read_text().strip() == digest and not force:
        return LIB
    srcs = [str(CSRC / s) for s in SOURCES if (CSRC / s).exists()]
    cmd = [nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared",
           "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
           "-I", str(ROOT / "include"), "-I", str(CSRC),
           "-DTF_BUILD_SO=1", *os.environ.get("TF_NVCC_EXTRA", "").split(),
           "-o", str(LIB) + ".tmp", *srcs]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        print(res.stderr, file=sys.stderr)
    os.replace(str(LIB) + ".tmp", LIB)
    stamp.write_text(digest + "\n")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
