"""Build the sm_100a C-ABI library in-tree (nvcc cross-compiles without a GPU).

Output: ``paper_2605_24832_b200/_lib/liboptimus_b200.so`` — travels to the GPU
box with the repo snapshot (git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "liboptimus_b200.so"
SOURCES = ["kv_append.cu", "paged_attn.cu", "unmask.cu", "capi.cu", "host_step.cu", "device_step.cu", "lmhead_unmask.cu"]
HEADERS = ["ptx.cuh", "attn.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3",
    "-Xcompiler",
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler",
    "-fPIC",
    "-Xptxas",
    "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "optimus_b200.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    LIBDIR.mkdir(exist_ok=True)
    objs = []
    logs = []
    for src in SOURCES:
        obj = LIBDIR / (Path(src).stem + ".o")
        cmd = [nvcc(), *ARCH, *FLAGS, "-I", str(PKG.parent / "include"), "-c", str(CSRC / src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(res.stderr)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(str(obj))
    tmp = LIBDIR / (LIB.name + ".tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    (LIBDIR / "ptxas.log").write_text("".join(logs))
    for o in objs:
        Path(o).unlink(missing_ok=True)
    if verbose:
        print("".join(logs))
    return LIB


REF_SRC = Path("/root/reference/pkg")
REF_DST = PKG.parent / "baseline" / "_ref"


def install_reference() -> bool:
    """Offline install of the reference package (``dllmsim``, pure Python) into
    ``baseline/_ref`` — git-ignored, but it travels to the GPU box with the snapshot,
    where the tests drive it with the B200 oracle plugged into ``Scenario.oracle_factory``
    (sim.py:64).  The checkout is read-only, so the install builds from a /tmp copy.
    Returns False when the checkout is absent (GPU box: the shipped install is used)."""
    if not REF_SRC.exists():
        return False
    tmp = Path("/tmp/optimus_refpkg")
    shutil.rmtree(tmp, ignore_errors=True)
    shutil.copytree(REF_SRC, tmp, ignore=shutil.ignore_patterns("tests", "test_output.txt", "__pycache__"))
    shutil.rmtree(REF_DST, ignore_errors=True)
    cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
           "--find-links", "/opt/wheelhouse", "--target", str(REF_DST), str(tmp), "-q"]
    subprocess.run(cmd, check=True)
    shutil.rmtree(tmp, ignore_errors=True)
    return True


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)
