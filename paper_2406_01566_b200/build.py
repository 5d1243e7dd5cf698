"""In-tree build of the engine (sm_100a) and the drop-in bindings.

Outputs (git-ignored, shipped to the GPU box by gpurun):
  paper_2406_01566_b200/lib/libhelio_gpu.so   C ABI (include/helio_gpu.h): kernels + K0
  paper_2406_01566_b200/lib/libhelio.so       C++ drop-in (namespace helio) over the C ABI
  paper_2406_01566_b200/_helio*.so            Python bindings (`_helio`)
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
OBJ = os.path.join(ROOT, "build", "obj")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v", "--expt-relaxed-constexpr"]
CXX_FLAGS = ["-O2", "-std=c++20", "-fPIC", "-ffp-contract=off", "-Wall", "-Wno-sign-compare"]

CU_SOURCES = ["helio_gpu.cu", "route.cu", "search.cu", "split.cu", "multi.cu"]
SHIM_SOURCES = ["shim_cluster.cpp", "shim_flow.cpp", "shim_plan.cpp", "shim_sched.cpp", "shim_heuristics.cpp"]
HEADERS = ["engine.h", "gen.h", "device_common.cuh", "build.cuh", "solve_parity.cuh", "solve_score.cuh", "shim.hpp",
           "shim_engine.hpp", "helio/cluster.hpp", "helio/errors.hpp", "helio/flow_graph.hpp", "helio/placement.hpp",
           "helio/scheduler.hpp", "helio/heuristics.hpp", "helio/rng.hpp"]


def _run(cmd, quiet=False):
    if not quiet:
        print("+", " ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} ... ({r.returncode})")
    return r.stdout + r.stderr


def _newer(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def ext_suffix() -> str:
    return sysconfig.get_config_var("EXT_SUFFIX") or ".so"


def build(force: bool = False, verbose: bool = False) -> None:
    os.makedirs(LIB, exist_ok=True)
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "helio_gpu.h")]
    objs = []
    ptxas_log = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        if force or _newer(o, [s] + hdrs):
            ptxas_log.append(_run([NVCC, *ARCH, *NVCC_FLAGS, "-c", s, "-o", o], quiet=not verbose))
        objs.append(o)
    libgpu = os.path.join(LIB, "libhelio_gpu.so")
    if force or _newer(libgpu, objs):
        # NCCL (the ranked argmax's all-gather) is bound at run time
        # (multi.cu nccl_api), never linked: torch needs its own newer copy
        _run([NVCC, *ARCH, "-shared", "-o", libgpu, *objs, "-lcudart_static", "-ldl"], quiet=not verbose)
    if ptxas_log:
        with open(os.path.join(ROOT, "build", "ptxas.log"), "w") as f:
            f.write("\n".join(ptxas_log))

    import pybind11  # noqa: WPS433 (build-time only)

    inc = ["-I" + CSRC, "-I" + os.path.join(ROOT, "include")]
    libshim = os.path.join(LIB, "libhelio.so")
    shim_srcs = [os.path.join(CSRC, f) for f in SHIM_SOURCES]
    if force or _newer(libshim, shim_srcs + [libgpu] + hdrs):
        _run(["g++", *CXX_FLAGS, *inc, "-shared", *shim_srcs, "-o", libshim,
              "-L" + LIB, "-lhelio_gpu", "-Wl,-rpath,$ORIGIN"], quiet=not verbose)
    pyext = os.path.join(PKG, "_helio" + ext_suffix())
    py_src = os.path.join(CSRC, "pymodule.cpp")
    if force or _newer(pyext, [py_src, libshim] + hdrs):
        _run(["g++", *CXX_FLAGS, *inc, "-I" + pybind11.get_include(),
              "-I" + sysconfig.get_paths()["include"], "-shared", py_src, "-o", pyext,
              "-L" + LIB, "-lhelio", "-lhelio_gpu", "-Wl,-rpath,$ORIGIN/lib"], quiet=not verbose)


# The reference's host planner + simulator, compiled from its own sources where
# they lie, linked over this drop-in's flow-graph and scheduler translation
# units (include/helio_planner.h).  Skipped, keeping a prebuilt library, when
# the reference tree is absent (the GPU box).
REF = os.environ.get("HELIO_REFERENCE", "/root/reference/proj")
PLANNER_REF_SOURCES = ["log", "cluster", "lp", "lp_format", "bnb", "heuristics", "placement", "workload", "sim"]
PLANNER_SHIM_SOURCES = ["shim_flow.cpp", "shim_sched.cpp"]


def _json_include() -> str:
    """nlohmann/json v3.11.3 single header (the reference vendors it but does not
    ship it, proj/.gitignore:2); the cudnn_frontend wheel carries the same file."""
    site = sysconfig.get_paths()["purelib"]
    return os.path.join(site, "include", "cudnn_frontend", "thirdparty", "nlohmann")


def build_planner(force: bool = False, verbose: bool = False) -> None:
    out = os.path.join(LIB, "libhelio_planner.so")
    if not os.path.exists(os.path.join(REF, "src", "sim.cpp")):
        if not verbose:
            return
        print(f"planner: {REF} absent; keeping prebuilt {out}" if os.path.exists(out) else
              f"planner: {REF} absent; plan(method='milp') and simulate() are unavailable")
        return
    pobj = os.path.join(OBJ, "planner")
    os.makedirs(pobj, exist_ok=True)
    ref_flags = ["-O3", "-DNDEBUG", "-std=c++20", "-fPIC", "-fvisibility=hidden", "-I" + os.path.join(REF, "include"),
                 "-I" + _json_include()]
    objs = []
    for name in PLANNER_REF_SOURCES:
        src = os.path.join(REF, "src", name + ".cpp")
        o = os.path.join(pobj, name + ".o")
        if force or _newer(o, [src]):
            _run(["g++", *ref_flags, "-c", src, "-o", o], quiet=not verbose)
        objs.append(o)
    api = os.path.join(CSRC, "planner", "planner_api.cpp")
    o = os.path.join(pobj, "planner_api.o")
    if force or _newer(o, [api, os.path.join(ROOT, "include", "helio_planner.h")]):
        _run(["g++", *ref_flags, "-c", api, "-o", o], quiet=not verbose)
    objs.append(o)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "helio_gpu.h")]
    for name in PLANNER_SHIM_SOURCES:
        src = os.path.join(CSRC, name)
        o = os.path.join(pobj, name.replace(".cpp", ".o"))
        if force or _newer(o, [src] + hdrs):
            _run(["g++", *CXX_FLAGS, "-fvisibility=hidden", "-I" + CSRC, "-I" + os.path.join(ROOT, "include"),
                  "-c", src, "-o", o], quiet=not verbose)
        objs.append(o)
    vs = os.path.join(OBJ, "planner", "exports.map")
    with open(vs, "w") as f:
        f.write("{ global: helio_planner_*; local: *; };\n")
    libgpu = os.path.join(LIB, "libhelio_gpu.so")
    if force or _newer(out, objs + [libgpu]):
        _run(["g++", "-shared", *objs, "-o", out, "-L" + LIB, "-lhelio_gpu", "-Wl,-rpath,$ORIGIN",
              "-Wl,--version-script=" + vs, "-lpthread"], quiet=not verbose)


def build_oracle() -> None:
    """Test infrastructure: oracle/_ref (reference, when /root/reference exists) + C oracle."""
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8"], quiet=True)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    build_planner(force="--force" in sys.argv, verbose=True)
    build_oracle()
