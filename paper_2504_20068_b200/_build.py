"""Build libjitsched.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libjitsched.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# two translation units: abi.cu (host code + the scoring kernel) and exact.cu (the resolve
# kernels and the exact radix path); both whole-program, no device-side launches
BASE = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "--fmad=false",
        "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
UNITS = [("abi.cu", []), ("exact.cu", [])]
LINK = ["-shared", "-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*")) + [os.path.join(ROOT, "include", "jit_sched.h")])


def build_library(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Build the library at `out` (default: the in-tree libjitsched.so); `defines` are extra -D
    flags for tuning experiments (profiles/variants.sh builds variants beside the default)."""
    newest = max(os.path.getmtime(s) for s in sources())
    if not force and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    tmp = out + f".tmp{os.getpid()}"
    inc = ["-I", os.path.join(ROOT, "include")]
    objs, log = [], ""
    try:
        for src, extra in UNITS:
            obj = tmp + "." + src + ".o"
            objs.append(obj)
            cmd = [NVCC] + BASE + extra + list(defines) + inc + ["-c", "-o", obj, os.path.join(HERE, "csrc", src)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src}:\n" + r.stdout[-4000:] + r.stderr[-8000:])
            log += r.stderr
        r = subprocess.run([NVCC] + LINK + ["-o", tmp] + objs, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + r.stdout[-4000:] + r.stderr[-8000:])
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    if verbose:
        print(log[-6000:])
    os.replace(tmp, out)
    return out
