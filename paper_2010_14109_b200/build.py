"""Build liboocore.so in-tree: host C++ (graph, planner, replay, runtime) and
CUDA kernels for sm_100a, linked with the static CUDA runtime so the library
loads on a machine without a GPU.

    python -m paper_2010_14109_b200.build        # incremental
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(os.path.dirname(HERE), "include")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "liboocore.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-I", INC, "-I", CSRC, "-Xcompiler", "-fPIC,-fvisibility=hidden",
          "-lineinfo"]


def _sources():
    out = []
    for root, _, files in os.walk(CSRC):
        for f in sorted(files):
            if f.endswith((".cpp", ".cu")):
                out.append(os.path.join(root, f))
    return sorted(out)


def _headers():
    hs = [os.path.join(INC, "oocore.h")]
    for root, _, files in os.walk(CSRC):
        hs += [os.path.join(root, f) for f in files if f.endswith((".hpp", ".cuh", ".h"))]
    return hs


def _compile(src, hdr_mtime, verbose):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    obj = os.path.join(OBJ, rel + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return obj, None
    cmd = [NVCC] + COMMON + ARCH
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if verbose else []
    else:
        cmd += ["-x", "cu"] if False else []
    cmd += ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        return obj, f"$ {' '.join(cmd)}\n{r.stdout}\n{r.stderr}"
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj, None


def build(verbose=False, jobs=None):
    os.makedirs(OBJ, exist_ok=True)
    hdr_mtime = max(os.path.getmtime(h) for h in _headers())
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=jobs or os.cpu_count()) as ex:
        res = list(ex.map(lambda s: _compile(s, hdr_mtime, verbose), srcs))
    errs = [e for _, e in res if e]
    if errs:
        raise RuntimeError("liboocore build failed:\n" + "\n".join(errs))
    objs = [o for o, _ in res]
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-ldl", "-lpthread", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n$ {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
