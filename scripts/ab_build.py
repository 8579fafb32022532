"""Build variants of libgreenllm.so for same-box A/B timing (kernel experiments).

Each variant is a list of (old, new) source replacements applied to a copy of
paper_2412_20322_b200/csrc; the result goes to build/ab/<name>.so.  Time them
with  GL_LIB_PATH=build/ab/<name>.so python scripts/quick_times.py ...

usage: python scripts/ab_build.py [variant ...]   (default: all in VARIANTS)
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2412_20322_b200", "csrc")
OUT = os.path.join(ROOT, "build", "ab")
sys.path.insert(0, ROOT)
from scripts.ab_variants import VARIANTS  # noqa: E402


def build(name, edits):
    tmp = os.path.join("/tmp", f"ab_{name}")
    shutil.rmtree(tmp, ignore_errors=True)
    shutil.copytree(SRC, tmp)
    for fname, old, new in edits:
        p = os.path.join(tmp, fname)
        s = open(p).read()
        assert s.count(old) == 1, (name, fname, old[:60], s.count(old))
        open(p, "w").write(s.replace(old, new))
    os.makedirs(OUT, exist_ok=True)
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
           "-o", os.path.join(OUT, f"{name}.so"), os.path.join(tmp, "greenllm.cu")]
    cmd[1:1] = os.environ.get("AB_FLAGS", "").split()  # e.g. AB_FLAGS="-Xptxas -O2"
    subprocess.check_call(cmd)
    print("built", name)


names = sys.argv[1:] or list(VARIANTS)
for n in names:
    base_name = n.split("@")[0]  # "<variant>@<tag>": the same edits under AB_FLAGS
    build(n, VARIANTS[base_name])
