"""Build libmppi_b200.so in-tree with nvcc for sm_100a (cross-compiles without a GPU)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmppi_b200.so")


def nccl_dirs():
    import nvidia.nccl as n  # torch wheel's NCCL (2.28.x); avoid the system 2.27 copy
    base = os.path.dirname(n.__file__) if getattr(n, "__file__", None) else list(n.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "mppi.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, trace: bool = False, extra: tuple = (), suffix: str = "") -> str:
    """trace=True builds the debug variant libmppi_b200_trace.so (-DMPPI_TC_TRACE kernel timeline)."""
    lib_out = LIB.replace(".so", ("_trace" if trace else "") + suffix + ".so")
    if os.environ.get("MPPI_SKIP_BUILD") == "1" and not force:   # development runs against MPPI_LIB
        return lib_out
    if not force and not trace and not suffix and not needs_build():
        return LIB
    inc, lib = nccl_dirs()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    tmp = lib_out + f".{os.getpid()}.tmp"
    flags = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-Xcompiler", "-fPIC",
             "-Xptxas", "-v" if verbose else "-O3", "-I", inc, "-I", os.path.join(ROOT, "include"),
             *(["-DMPPI_TC_TRACE"] if trace else []), *extra]
    # one nvcc per translation unit, in parallel (the two tensor-core kernels dominate), then one link
    objs = [f"{tmp}.{os.path.basename(src)}.o" for src in sources()]

    # per-TU object cache (local builds only): key = the TU, every header it can include, the flags
    import hashlib, shutil
    cache = os.environ.get("MPPI_OBJ_CACHE", "/tmp/mppi_objcache")
    hdrs = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "mppi.h")]
    hdr_hash = hashlib.sha256(b"".join(open(h, "rb").read() for h in hdrs) + " ".join(flags).encode()).hexdigest()

    def compile_one(src_obj):
        src, obj = src_obj
        key = hashlib.sha256(open(src, "rb").read() + hdr_hash.encode()).hexdigest()[:24]
        cached = os.path.join(cache, f"{os.path.basename(src)}.{key}.o")
        try:
            if os.path.exists(cached) and not verbose:
                shutil.copyfile(cached, obj)
                return subprocess.CompletedProcess([], 0, "", "")
        except OSError:
            pass
        r = subprocess.run([nvcc, *flags, "-c", src, "-o", obj], capture_output=True, text=True)
        if r.returncode == 0:
            try:   # the cache is an optimisation only
                os.makedirs(cache, exist_ok=True)
                shutil.copyfile(obj, cached + f".{os.getpid()}")
                os.replace(cached + f".{os.getpid()}", cached)
            except OSError:
                pass
        return r
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(objs)) as ex:
        results = list(ex.map(compile_one, zip(sources(), objs)))
    r = None
    for res in results:
        if verbose or res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
    if all(res.returncode == 0 for res in results):
        r = subprocess.run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-L", lib,
                            "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}", "-o", tmp], capture_output=True, text=True)
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    if r is None or r.returncode != 0:
        if r is not None:
            sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc build of libmppi_b200.so failed")
    os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    ex = tuple(a for a in sys.argv[1:] if a.startswith("-D"))
    sfx = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--suffix=")), "")
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv, extra=ex, suffix=sfx))
