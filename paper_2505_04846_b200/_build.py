"""Build the in-tree shared libraries with nvcc for sm_100a (no GPU needed to build).

* paper_2505_04846_b200/libhiper.so  -- the product: C ABI of include/hiper.h (CUDA kernels + host)
* synth/libsynth.so                  -- the device side of the seeded input generator (test/bench)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2505_04846_b200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-shared", "-Xcompiler", "-fPIC", "-Xcompiler",
          "-fvisibility=hidden", "--expt-relaxed-constexpr"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        inc, lib = os.path.join(base, "nccl", "include"), os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    raise RuntimeError("pip NCCL (nvidia-nccl-cu12, the one torch loads) not found")


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed: " + " ".join(cmd))
    return r.stdout + r.stderr


def build_hiper(force=False, verbose=False, debug=False) -> str:
    """libhiper.so; debug=True: libhiper_debug.so with the device-side checks (HIPER_DASSERT)."""
    out = os.path.join(PKG, "libhiper_debug.so" if debug else "libhiper.so")
    srcs = (glob.glob(os.path.join(PKG, "csrc", "**", "*.cu*"), recursive=True)
            + [os.path.join(ROOT, "include", "hiper.h")])
    if force or _stale(out, srcs):
        inc, lib = nccl_dirs()
        tmp = out + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, *COMMON, "-I", os.path.join(ROOT, "include"), "-I", inc,
               "-DHIPER_BUILD", *(["-DHIPER_DEVICE_ASSERTS"] if debug else []),
               os.path.join(PKG, "csrc", "hiper_api.cu"), "-o", tmp,
               "-L", lib, "-l:libnccl.so.2", f"-Xlinker=-rpath,{lib}"]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        log = _run(cmd)
        if verbose:
            print(log)
        os.replace(tmp, out)
    return out


def build_synth(force=False) -> str:
    out = os.path.join(ROOT, "synth", "libsynth.so")
    src = os.path.join(ROOT, "synth", "csrc", "synth.cu")
    if force or _stale(out, [src]):
        tmp = out + f".tmp{os.getpid()}"
        _run([NVCC, *ARCH, *COMMON, src, "-o", tmp])
        os.replace(tmp, out)
    return out


def build_all(force=False, verbose=False):
    """The product library, its device-assert twin and the generator, compiled concurrently."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(3) as ex:
        jobs = [ex.submit(build_hiper, force, verbose), ex.submit(build_hiper, force, False, True),
                ex.submit(build_synth, force)]
        return tuple(j.result() for j in jobs)


if __name__ == "__main__":
    print(build_all(force="--force" in sys.argv, verbose="-v" in sys.argv))
