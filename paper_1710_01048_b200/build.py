"""In-tree build of libwgq.so (sm_100a) with nvcc.

    python -m paper_1710_01048_b200.build        # or __graft_entry__.build()
"""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libwgq.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["rules.cpp", "api.cpp", "host_pipeline.cpp", "tables.cu", "assemble.cu", "assemble_line.cu", "fourier2d.cu", "separable.cu", "grid.cu", "checks.cu"]
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "--expt-relaxed-constexpr"]


def sources():
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "wgq.h")]
    return all(os.path.getmtime(d) <= t for d in deps)


def write_build_info():
    """paper_1710_01048_b200/build_info.json: the git commit the library was built from (the GPU
    box receives a snapshot without .git; bench.py reports it)."""
    import json
    import time
    info = {"built": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    try:
        sha = subprocess.run(["git", "-C", ROOT, "rev-parse", "HEAD"], capture_output=True, text=True, timeout=10)
        dirty = subprocess.run(["git", "-C", ROOT, "status", "--porcelain", "--untracked-files=no"],
                               capture_output=True, text=True, timeout=10)
        if sha.returncode == 0:
            info["git_sha"] = sha.stdout.strip()
            info["dirty"] = bool(dirty.stdout.strip())
    except Exception:
        pass
    with open(os.path.join(PKG, "build_info.json"), "w") as f:
        json.dump(info, f)


def build(force=False, verbose=False):
    if not force and up_to_date():
        write_build_info()
        return LIB
    objs = []
    os.makedirs(os.path.join(PKG, "build"), exist_ok=True)
    for src in sources():
        obj = os.path.join(PKG, "build", os.path.basename(src) + ".o")
        cmd = [NVCC] + FLAGS + ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(obj)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB] + objs + ["-lcudart"]
    subprocess.run(cmd, check=True)
    write_build_info()
    # peak microbenchmarks (write-only HBM, copy, DFMA) used by bench.py's extras
    peaks_src = os.path.join(ROOT, "tools", "peaks.cu")
    if os.path.exists(peaks_src):                 # optional tool: a failure here never fails the build
        subprocess.run([NVCC, "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o",
                        os.path.join(ROOT, "tools", "peaks"), peaks_src], check=False)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
