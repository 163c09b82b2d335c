"""Build libwgq with an alternative source for one file (kernel experiments).

    python tools/build_variant.py NAME path/to/assemble_line.cu [more overrides...]

Writes variants/NAME.so (git-ignored; travels to the GPU box with gpurun); select it with
WGQ_LIB=variants/NAME.so.  Each override replaces the csrc file of the same basename.
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1710_01048_b200 import build as B  # noqa: E402

name, overrides = sys.argv[1], sys.argv[2:]
tmp = tempfile.mkdtemp()
csrc = os.path.join(tmp, "csrc")
shutil.copytree(B.CSRC, csrc)
for o in overrides:
    shutil.copy(o, os.path.join(csrc, os.path.basename(o)))
objs = []
for src in B.SOURCES:
    obj = os.path.join(tmp, src + ".o")
    subprocess.run([B.NVCC] + B.FLAGS + ["-I", os.path.join(ROOT, "include"), "-I", csrc, "-c",
                    os.path.join(csrc, src), "-o", obj], check=True)
    objs.append(obj)
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
out = os.path.join(ROOT, "variants", name + ".so")
subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out] + objs + ["-lcudart"],
               check=True)
print(out)
