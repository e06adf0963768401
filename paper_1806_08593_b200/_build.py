"""Build libtmc.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "tmc_api.cu")
OUT = os.path.join(HERE, "libtmc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "128"]


def sources():
    return [SRC] + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + glob.glob(os.path.join(HERE, "csrc", "*.h")) \
        + [os.path.join(ROOT, "include", "tmc.h")]


def build_variant(name: str, defines, verbose: bool = False) -> str:
    """An experiment variant of the library (e.g. libtmc_spin.so with -DTMC_SPIN_WAIT)."""
    out = os.path.join(HERE, f"libtmc_{name}.so")
    cmd = [NVCC] + FLAGS + [f"-D{d}" for d in defines] + ["-o", out, SRC]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return out


def build_debug(force: bool = False, verbose: bool = False) -> str:
    """libtmc_debug.so: the release library plus an mbarrier-wait deadline (-DTMC_DEBUG_SYNC): a lost
    pipeline phase traps with the barrier's address instead of hanging the GPU."""
    out = os.path.join(HERE, "libtmc_debug.so")
    if not force and os.path.exists(out) and all(os.path.getmtime(s) <= os.path.getmtime(out) for s in sources()):
        return out
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC] + FLAGS + ["-DTMC_DEBUG_SYNC", "-o", tmp, SRC]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


def build_instrumented(verbose: bool = False) -> str:
    """libtmc_instr.so: the same library with per-CTA barrier-wait counters (experiments only)."""
    out = os.path.join(HERE, "libtmc_instr.so")
    if os.path.exists(out) and all(os.path.getmtime(s) <= os.path.getmtime(out) for s in sources()):
        return out
    cmd = [NVCC] + FLAGS + ["-DTMC_INSTRUMENT", "-o", out, SRC]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(OUT):
        t = os.path.getmtime(OUT)
        if all(os.path.getmtime(s) <= t for s in sources()):
            return OUT
    tmp = OUT + f".tmp{os.getpid()}"
    cmd = [NVCC] + FLAGS + ["-o", tmp, SRC]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force=True, verbose=True)
