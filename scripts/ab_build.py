"""Build A/B variants of libgreenllm.so for same-box timing (kernel experiments).

A variant is the tree's csrc/ with some -D macro settings (e.g. GL_SAT2_MIN in older
revisions) or a patch file of (old, new) replacements; the result goes to
build/ab/<name>.so.  Time variants with  scripts/ab_times.sh <name>...

    python scripts/ab_build.py <name> [-Dmacro=value ...] [--patch file.py]

A patch file defines EDITS = [(csrc file name, old text, new text), ...].  The
round-2 experiments and their outcomes are in profiles/r02_decode_ab.md; their
sources are in the git history of k_decode.cuh.
"""
import os
import runpy
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2412_20322_b200", "csrc")
OUT = os.path.join(ROOT, "build", "ab")


def build(name, defines=(), edits=()):
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
           "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"), *defines,
           "-o", os.path.join(OUT, f"{name}.so"), os.path.join(tmp, "greenllm.cu")]
    subprocess.check_call(cmd)
    print("built", name)


if __name__ == "__main__":
    args = sys.argv[1:]
    if not args:
        sys.exit(__doc__)
    name, rest = args[0], args[1:]
    defines = [a for a in rest if a.startswith("-D")]
    edits = []
    if "--patch" in rest:
        edits = runpy.run_path(rest[rest.index("--patch") + 1])["EDITS"]
    build(name, defines, edits)
