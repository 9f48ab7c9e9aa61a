"""In-tree build of the native libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

  libgss.so           CUDA kernels + C ABI (include/gss.h), sm_100a
  _survscan*.so       pybind11 module: the reference's Python API over the
                      C++ mirror of survscan::{Engine, fit, cross_validate, ...}

    python -m paper_2204_08183_b200.build [--force]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBGSS = os.environ.get("GSS_LIB") or os.path.join(PKG, "libgss.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _newer(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build_libgss(force=False):
    """Each .cu compiles to its own object (in parallel, only when it or a
    shared header changed), then one link."""
    from concurrent.futures import ThreadPoolExecutor
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "gss.h")]
    extra = ["-DGSS_ENABLE_TRACE=1"] if os.environ.get("GSS_TRACE_BUILD") == "1" else []
    objdir = os.path.join(ROOT, "build", "obj" + ("_trace" if extra else ""))
    os.makedirs(objdir, exist_ok=True)
    objs, todo = [], []
    for src in cu:
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + hdrs):
            todo.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                         "-diag-suppress", "177", *extra, "-c", src, "-o", obj])
    with ThreadPoolExecutor(max(1, len(todo))) as ex:
        list(ex.map(_run, todo))
    if force or todo or _newer(LIBGSS, objs):
        _run([NVCC, *ARCH, "-shared", *objs, "-o", LIBGSS])
    return LIBGSS


def ext_path():
    return os.path.join(PKG, "_survscan" + sysconfig.get_config_var("EXT_SUFFIX"))


LIBSURVSCAN = os.path.join(PKG, "libsurvscan_b200.so")


def build_libsurvscan(force=False):
    """C++ mirror of the reference API (namespace survscan) over libgss."""
    host = os.path.join(CSRC, "host")
    srcs = sorted(s for s in glob.glob(os.path.join(host, "*.cpp"))
                  if not s.endswith("bindings.cpp"))
    deps = srcs + glob.glob(os.path.join(host, "survscan", "*.hpp")) + [LIBGSS]
    if force or _newer(LIBSURVSCAN, deps):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-pthread",
              "-I" + host, *srcs, "-L" + PKG, "-lgss", "-Wl,-rpath,$ORIGIN",
              "-o", LIBSURVSCAN])
    return LIBSURVSCAN


def build_pymodule(force=False):
    """pybind11 `_survscan`: the reference's Python API over libsurvscan_b200."""
    host = os.path.join(CSRC, "host")
    src = os.path.join(host, "bindings.cpp")
    deps = [src, LIBSURVSCAN] + glob.glob(os.path.join(host, "survscan", "*.hpp"))
    out = ext_path()
    if force or _newer(out, deps):
        import pybind11
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-pthread",
              "-I" + host, "-I" + sysconfig.get_paths()["include"], "-I" + pybind11.get_include(),
              src, "-L" + PKG, "-lsurvscan_b200", "-lgss", "-Wl,-rpath,$ORIGIN", "-o", out])
    return out


def build(force=False):
    build_libgss(force)
    build_libsurvscan(force)
    build_pymodule(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
