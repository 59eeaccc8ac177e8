"""Build an A/B variant of libcc from a modified copy of csrc/ (development tool):
    python tools/build_variant.py NAME 'python-expr-on-(path, text)' ...
Each edit is "FILE::OLD::NEW" (literal replace); the variant lands in variants/libcc_NAME.so
(in-tree so it travels to the GPU box; load it with CC_LIB_PATH)."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_18801_b200 import build as B  # noqa: E402

name = sys.argv[1]
src = os.path.join(ROOT, "paper_2604_18801_b200", "csrc")
base = f"/tmp/cc_variant_{name}"
shutil.rmtree(base, ignore_errors=True)
work = os.path.join(base, "pkg", "csrc")
shutil.copytree(src, work)
shutil.copytree(os.path.join(ROOT, "include"), os.path.join(base, "include"))  # csrc includes ../../include/cc.h
for spec in sys.argv[2:]:
    f, old, new = spec.split("::")
    p = os.path.join(work, f)
    s = open(p).read()
    assert old in s, (f, old[:60])
    open(p, "w").write(s.replace(old, new))
out = os.path.join(ROOT, "variants")
os.makedirs(out, exist_ok=True)
objs = []
for cu in sorted(x for x in os.listdir(work) if x.endswith(".cu")):
    o = os.path.join(work, cu[:-3] + ".o")
    subprocess.check_call([B.NVCC, *B.ARCH, *[x for x in B.FLAGS if x != "-Xptxas" and x != "-warn-spills"],
                           f"-I{work}", "-c", os.path.join(work, cu), "-o", o])
    objs.append(o)
lib = os.path.join(out, f"libcc_{name}.so")
subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, *B.LDFLAGS])
print(lib)
