"""Build the C-ABI library of another git revision into tools/_bin/lib_<rev>.so, for
same-process A/B timing against the working tree (tools/ab_lib.py).

    python tools/build_variant.py HEAD
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2605_24832_b200 import build as B  # noqa: E402

rev = sys.argv[1] if len(sys.argv) > 1 else "HEAD"
sha = subprocess.check_output(["git", "rev-parse", "--short", rev], cwd=ROOT, text=True).strip()
out = ROOT / "tools" / "_bin" / f"src_{sha}"
(out / "paper_2605_24832_b200" / "csrc").mkdir(parents=True, exist_ok=True)
(out / "include").mkdir(parents=True, exist_ok=True)
files = subprocess.check_output(["git", "ls-tree", "--name-only", rev, "paper_2605_24832_b200/csrc/", "include/"],
                                cwd=ROOT, text=True).split()
for f in files:
    (out / f).write_bytes(subprocess.check_output(["git", "show", f"{rev}:{f}"], cwd=ROOT))
csrc = out / "paper_2605_24832_b200" / "csrc"
objs = []
for src in sorted(csrc.glob("*.cu")):
    obj = csrc / (src.stem + ".o")
    subprocess.run([B.nvcc(), *B.ARCH, *[f for f in B.FLAGS if f != "-v" and f != "-Xptxas"], "-I", str(out / "include"),
                    "-c", str(src), "-o", str(obj)], check=True)
    objs.append(str(obj))
lib = ROOT / "tools" / "_bin" / f"lib_{sha}.so"
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(lib), *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"],
               check=True)
print(lib)
