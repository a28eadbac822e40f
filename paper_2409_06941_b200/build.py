"""In-tree build of the product library `_lib/libfreeride.so`.

Host C++ (csrc/host, csrc/capi_*.cpp, csrc/runtime) is compiled with g++
(C++20, -O2, -ffp-contract=off so host doubles match the reference bit for
bit); device code (csrc/kernels/*.cu) with nvcc for sm_100a only
(`-gencode arch=compute_100a,code=sm_100a -lineinfo`).  cudart is linked
statically so the library carries its own runtime next to torch's.  Objects
are rebuilt when a source or any header under csrc/ or include/ is newer.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
OBJ = os.path.join(os.path.dirname(HERE), "build", "obj")
OUT = os.path.join(HERE, "_lib", "libfreeride.so")
SIM = os.path.join(HERE, "_lib", "freeride-sim")  # the CLI (csrc/tools, host objects only)
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = [f"-I{INCLUDE}", f"-I{CSRC}", f"-I{CUDA}/include"]
CXXFLAGS = ["-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-Wall", "-Wextra",
            "-Wno-unused-parameter", "-pthread"]
NVCCFLAGS = ["-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC",
             "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _sources():
    cpp = sorted(p for p in glob.glob(os.path.join(CSRC, "**", "*.cpp"), recursive=True)
                 if os.sep + "tools" + os.sep not in p)
    cu = sorted(glob.glob(os.path.join(CSRC, "**", "*.cu"), recursive=True))
    return cpp, cu


def _headers_mtime():
    hs = glob.glob(os.path.join(CSRC, "**", "*.h*"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
    hs += glob.glob(os.path.join(INCLUDE, "*.h"))
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def _obj_for(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "__")
    return os.path.join(OBJ, rel + ".o")


def _stale(src, obj, hdr_mtime):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return os.path.getmtime(src) > t or hdr_mtime > t


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


def build(verbose: bool = False, jobs: int = 0) -> str:
    if not os.path.exists(NVCC):
        raise RuntimeError(f"nvcc not found at {NVCC}")
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cpp, cu = _sources()
    hm = _headers_mtime()
    cmds = []
    for s in cpp:
        o = _obj_for(s)
        if _stale(s, o, hm):
            cmds.append([os.environ.get("CXX", "g++"), *CXXFLAGS, *INC, "-c", s, "-o", o])
    for s in cu:
        o = _obj_for(s)
        if _stale(s, o, hm):
            cmds.append([NVCC, *NVCCFLAGS, *INC, "-c", s, "-o", o])
    jobs = jobs or min(8, os.cpu_count() or 4)
    with ThreadPoolExecutor(jobs) as ex:
        for out in ex.map(_run, cmds):
            if verbose and out.strip():
                print(out)
    objs = [_obj_for(s) for s in cpp + cu]
    if not os.path.exists(OUT) or cmds or any(os.path.getmtime(o) > os.path.getmtime(OUT)
                                              for o in objs):
        tmp = OUT + ".tmp"
        _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static",
              f"-L{CUDA}/lib64", "-lcublasLt", "-Xlinker", f"-rpath={CUDA}/lib64",
              "-Xcompiler", "-pthread"])
        shutil.move(tmp, OUT)
    # the CLI: its own main + the pure-C++ host objects (no CUDA)
    tool = os.path.join(CSRC, "tools", "freeride_sim.cpp")
    tool_o = _obj_for(tool)
    cxx = os.environ.get("CXX", "g++")
    if _stale(tool, tool_o, hm):
        _run([cxx, *CXXFLAGS, *INC, "-c", tool, "-o", tool_o])
    host_objs = [_obj_for(s) for s in cpp if os.sep + "host" + os.sep in s]
    if not os.path.exists(SIM) or any(os.path.getmtime(o) > os.path.getmtime(SIM) for o in host_objs + [tool_o]):
        _run([cxx, "-o", SIM + ".tmp", tool_o, *host_objs, "-pthread"])
        shutil.move(SIM + ".tmp", SIM)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
