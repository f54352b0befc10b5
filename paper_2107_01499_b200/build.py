"""Build recipe for libb2comm.so (sm_100a) and librcomm_b200.so (C++ host layer).

Plain nvcc/g++ invocations, outputs in-tree next to this file so the built
libraries travel to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
HOST = os.path.join(PKG_DIR, "host")
INCLUDE = os.path.join(REPO, "include")
LIB = os.path.join(PKG_DIR, "libb2comm.so")
HOSTLIB = os.path.join(PKG_DIR, "librcomm_b200.so")

CUDA_SOURCES = ["codec.cu", "collectives.cu", "comm.cu", "onebit_coll.cu", "small_coll.cu", "central_stag.cu",
                "small_central.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _deps(dirpath: str, exts: tuple[str, ...]) -> list[str]:
    return [os.path.join(dirpath, f) for f in sorted(os.listdir(dirpath)) if f.endswith(exts)]


def build_variant(name: str, defines: list[str]) -> str:
    """A compile-time variant of libb2comm.so (e.g. -DB2_RING_STAGES=6) under
    variants/, selected at run time with B2COMM_LIB (A/B measurements)."""
    return build_cuda(force=False, out=os.path.join(PKG_DIR, "variants", f"libb2comm_{name}.so"),
                      extra=[f"-D{d}" for d in defines], objdir=os.path.join(PKG_DIR, "build", name))


def build_cuda(force: bool = False, verbose: bool = False, out: str | None = None, extra: list | None = None,
               objdir: str | None = None) -> str:
    LIB = out or globals()["LIB"]
    deps = _deps(CSRC, (".cu", ".cuh", ".h")) + [os.path.join(INCLUDE, "b2comm.h")]
    if not force and not _stale(LIB, deps):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    objdir = objdir or os.path.join(PKG_DIR, "build")
    os.makedirs(objdir, exist_ok=True)
    nvcc = _nvcc()
    objs = []
    for src in CUDA_SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc, *NVCC_FLAGS, *(extra or []), "-I", INCLUDE, "-I", CSRC, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        with open(os.path.join(objdir, src + ".ptxas.txt"), "w") as f:
            f.write(r.stderr)
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-Xlinker", "--exclude-libs,ALL"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    return LIB


def build_host(force: bool = False) -> str | None:
    """C++ host layer mirroring rcomm's API over the C ABI."""
    if not os.path.isdir(HOST):
        return None
    # rcomm_link.cpp is the link-time drop-in built against the REFERENCE's
    # headers (build_dropin), not part of this library
    srcs = [p for p in _deps(HOST, (".cpp",)) if not p.endswith("rcomm_link.cpp")]
    if not srcs:
        return None
    deps = srcs + _deps(os.path.join(INCLUDE, "rcomm_b200"), (".hpp",)) + [LIB]
    if not force and not _stale(HOSTLIB, deps):
        return HOSTLIB
    cuda_inc = "/usr/local/cuda/include"
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", INCLUDE, "-I", cuda_inc, *srcs,
           "-o", HOSTLIB + ".tmp", "-L", PKG_DIR, "-lb2comm", "-Wl,-rpath,$ORIGIN",
           "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed on the host layer")
    os.replace(HOSTLIB + ".tmp", HOSTLIB)
    return HOSTLIB


HOST_TEST_SRC = os.path.join(REPO, "tests", "cpp", "test_host_api.cpp")
HOST_TEST_BIN = os.path.join(REPO, "tests", "cpp", "test_host_api")


def build_host_test(force: bool = False) -> str | None:
    """C++ test of the drop-in layer (links the oracle as its checker)."""
    oracle_dir = os.path.join(REPO, "oracle")
    liboracle = os.path.join(oracle_dir, "liboracle.so")
    if not (os.path.exists(HOST_TEST_SRC) and os.path.exists(HOSTLIB) and os.path.exists(liboracle)):
        return None
    if not force and not _stale(HOST_TEST_BIN, [HOST_TEST_SRC, HOSTLIB, liboracle]):
        return HOST_TEST_BIN
    cmd = ["g++", "-std=c++20", "-O2", "-I", INCLUDE, "-I", "/usr/local/cuda/include", HOST_TEST_SRC,
           "-o", HOST_TEST_BIN + ".tmp", "-L", PKG_DIR, "-lrcomm_b200", "-lb2comm", "-L", oracle_dir, "-loracle",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lpthread",
           f"-Wl,-rpath,{PKG_DIR}:{oracle_dir}:/usr/local/cuda/lib64",
           "-Wl,-rpath,$ORIGIN/../../paper_2107_01499_b200:$ORIGIN/../../oracle"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed on the host-layer test")
    os.replace(HOST_TEST_BIN + ".tmp", HOST_TEST_BIN)
    return HOST_TEST_BIN


NVL_PROBE_SRC = os.path.join(REPO, "tests", "cpp", "nvl_probe.cpp")
NVL_PROBE_BIN = os.path.join(REPO, "tests", "cpp", "nvl_probe")


def build_nvl_probe(force: bool = False) -> str | None:
    """Dev probe: every GPU in one process (thread per GPU) running a
    primitive back to back, so ncu --devices 0 can count NVLink bytes."""
    if not (os.path.exists(NVL_PROBE_SRC) and os.path.exists(HOSTLIB)):
        return None
    if not force and not _stale(NVL_PROBE_BIN, [NVL_PROBE_SRC, HOSTLIB, LIB]):
        return NVL_PROBE_BIN
    cmd = ["g++", "-std=c++20", "-O2", "-I", INCLUDE, "-I", "/usr/local/cuda/include", NVL_PROBE_SRC,
           "-o", NVL_PROBE_BIN + ".tmp", "-L", PKG_DIR, "-lrcomm_b200", "-lb2comm", "-L/usr/local/cuda/lib64",
           "-lcudart", "-lpthread", "-Wl,-rpath,$ORIGIN/../../paper_2107_01499_b200",
           f"-Wl,-rpath,{PKG_DIR}:/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed on nvl_probe")
    os.replace(NVL_PROBE_BIN + ".tmp", NVL_PROBE_BIN)
    return NVL_PROBE_BIN


REF_PROJ = "/root/reference/proj"
DROPIN_SRC = os.path.join(REPO, "tests", "cpp", "algo_dropin.cpp")
DROPIN_REF_BIN = os.path.join(REPO, "tests", "cpp", "algo_dropin_ref")
DROPIN_B200_BIN = os.path.join(REPO, "tests", "cpp", "algo_dropin_b200")


def build_dropin(force: bool = False) -> tuple | None:
    """The reference's own algorithms.cpp (UNMODIFIED, compiled in place from
    /root/reference) linked twice: with its collectives.cpp on SimCluster
    (algo_dropin_ref) and with host/rcomm_link.cpp -- the B200 primitives
    behind the reference's API -- instead (algo_dropin_b200).  Needs the
    reference tree, so it is built here; the binaries travel to the GPU box
    with the snapshot.  Reference sources are never copied into the repo."""
    src = os.path.join(REF_PROJ, "src")
    if not (os.path.isdir(src) and os.path.exists(DROPIN_SRC) and os.path.exists(LIB)):
        return None
    link_cpp = os.path.join(HOST, "rcomm_link.cpp")
    common = ["algorithms.cpp", "kernels.cpp", "kernels_avx2.cpp", "tensor.cpp", "codec.cpp"]
    ref_only = ["collectives.cpp", "sim_transport.cpp"]
    deps = [DROPIN_SRC, link_cpp, LIB, os.path.join(INCLUDE, "rcomm_b200", "rcomm_link.hpp")] + \
        [os.path.join(src, f) for f in common + ref_only]
    if not force and not _stale(DROPIN_REF_BIN, deps) and not _stale(DROPIN_B200_BIN, deps):
        return DROPIN_REF_BIN, DROPIN_B200_BIN
    objdir = os.path.join(REPO, "tests", "cpp", "dropin_obj")
    os.makedirs(objdir, exist_ok=True)
    flags = ["g++", "-std=c++20", "-O2", "-g", "-I", os.path.join(REF_PROJ, "include")]  # CMakeLists.txt:3,9

    def obj(path, extra=()):
        o = os.path.join(objdir, os.path.basename(path).replace(".cpp", ".o"))
        if force or _stale(o, [path]):
            r = subprocess.run([*flags, *extra, "-c", path, "-o", o], capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"g++ failed on {path}")
        return o

    objs = [obj(os.path.join(src, f), ["-mavx2"] if f == "kernels_avx2.cpp" else []) for f in common]
    cuda = ["-I", INCLUDE, "-I", "/usr/local/cuda/include"]
    link_o = os.path.join(objdir, "rcomm_link.o")
    drv_b200 = os.path.join(objdir, "algo_dropin_b200.o")
    drv_ref = os.path.join(objdir, "algo_dropin_ref.o")
    for cmd in ([*flags, *cuda, "-c", link_cpp, "-o", link_o],
                [*flags, *cuda, "-c", DROPIN_SRC, "-o", drv_b200],
                [*flags, "-DDROPIN_REF", "-c", DROPIN_SRC, "-o", drv_ref]):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("g++ failed on the drop-in test")
    ref_objs = [obj(os.path.join(src, f)) for f in ref_only]
    for out, extra in ((DROPIN_REF_BIN, [drv_ref, *ref_objs]),
                       (DROPIN_B200_BIN, [drv_b200, link_o, "-L", PKG_DIR, "-lb2comm",
                                          "-L/usr/local/cuda/lib64", "-lcudart",
                                          f"-Wl,-rpath,{PKG_DIR}:/usr/local/cuda/lib64",
                                          "-Wl,-rpath,$ORIGIN/../../paper_2107_01499_b200"])):
        r = subprocess.run(["g++", "-o", out + ".tmp", *objs, *extra, "-lpthread"], capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"link failed for {out}")
        os.replace(out + ".tmp", out)
    return DROPIN_REF_BIN, DROPIN_B200_BIN


def build(force: bool = False, verbose: bool = False) -> None:
    build_cuda(force=force, verbose=verbose)
    build_host(force=force)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
