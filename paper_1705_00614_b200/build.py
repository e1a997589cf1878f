"""Build libswflood_cuda.so in-tree for sm_100a (nvcc, no JIT cache)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libswflood_cuda.so")
SOURCES = ["swf_capi.cu", "swf_stage.cu", "swf_fused.cu", "swf_nest.cu", "swf_free.cu"]
HEADERS = ["swf_math.cuh", "swf_internal.cuh"]

# -fmad=false: no FMA contraction, so every + and * rounds exactly like the
# reference's x86-64 build.
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-diag-suppress", "177",
]


def nvcc():
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if p and os.path.exists(p):
            return p
    return "nvcc"


def stale(out=OUT):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "swf.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


HOST_SRCS = [os.path.join(HERE, "host", f) for f in
             ("swflood_b200.cpp", "swflood_nest.cpp", "swflood_io.cpp")]
HOST_OUT = os.path.join(HERE, "libswflood_b200.so")
CLI_SRC = os.path.join(HERE, "host", "swflood_cli.cpp")
CLI_OUT = os.path.join(HERE, "swflood")
INCLUDE = os.path.join(HERE, "..", "include")


def _cxx():
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def build_host(force=False):
    """The C++ drop-in API (include/swflood_b200.hpp, include/swflood/*.hpp)
    over the C ABI, and the `swflood` command-line driver."""
    hdrs = [os.path.join(INCLUDE, "swflood_b200.hpp"), os.path.join(INCLUDE, "swf.h"),
            os.path.join(INCLUDE, "swflood", "nesting.hpp"), os.path.join(INCLUDE, "swflood", "io.hpp")]
    deps = HOST_SRCS + hdrs + [OUT]
    if force or not os.path.exists(HOST_OUT) or any(
            os.path.getmtime(d) > os.path.getmtime(HOST_OUT) for d in deps):
        cmd = [_cxx(), "-std=c++20", "-O2", "-fPIC", "-shared", "-I", INCLUDE] + HOST_SRCS + \
            ["-o", HOST_OUT, "-L", HERE, "-lswflood_cuda", "-Wl,-rpath,$ORIGIN"]
        subprocess.run(cmd, check=True)
    build_pybind(force, hdrs)
    if force or not os.path.exists(CLI_OUT) or any(
            os.path.getmtime(d) > os.path.getmtime(CLI_OUT) for d in [CLI_SRC, HOST_OUT] + hdrs):
        cmd = [_cxx(), "-std=c++20", "-O2", "-I", INCLUDE, CLI_SRC, "-o", CLI_OUT, "-L", HERE,
               "-lswflood_b200", "-lswflood_cuda", "-Wl,-rpath,$ORIGIN"]
        subprocess.run(cmd, check=True)
    return HOST_OUT


PYBIND_SRC = os.path.join(HERE, "host", "swflood_pybind.cpp")


def pybind_out():
    import sysconfig
    return os.path.join(HERE, "swflood_native" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_pybind(force=False, hdrs=()):
    """pybind11 module `swflood_native` over libswflood_b200.so (the
    reference's missing bindings/ directory); skipped if pybind11 is absent."""
    try:
        import pybind11
    except ImportError:
        return None
    import sysconfig
    out = pybind_out()
    deps = [PYBIND_SRC, HOST_OUT] + list(hdrs)
    if force or not os.path.exists(out) or any(os.path.getmtime(d) > os.path.getmtime(out) for d in deps):
        cmd = [_cxx(), "-std=c++20", "-O2", "-fPIC", "-shared", "-I", INCLUDE,
               "-I", pybind11.get_include(), "-I", sysconfig.get_paths()["include"], PYBIND_SRC,
               "-o", out, "-L", HERE, "-lswflood_b200", "-lswflood_cuda", "-Wl,-rpath,$ORIGIN"]
        subprocess.run(cmd, check=True)
    return out


def _compile_link(out, flags, objdir, verbose=False):
    """One nvcc process per translation unit (in parallel), then the link."""
    os.makedirs(objdir, exist_ok=True)
    procs, objs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc()] + flags + ["-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd, cwd=CSRC), cmd))
        objs.append(obj)
    bad = [c for p, c in procs if p.wait() != 0]
    if bad:
        raise subprocess.CalledProcessError(1, bad[0])
    subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out]
                   + objs, check=True, cwd=CSRC)


# The opt-in FAST build (include/swf.h swf_build_flavor): FMA contraction,
# CUDA's cbrt, reciprocal multiplications -- tolerance-validated, not bit-exact.
OUT_FAST = os.path.join(HERE, "libswflood_cuda_fast.so")
FAST_FLAGS = [f for f in NVCC_FLAGS if f != "-fmad=false"] + ["-fmad=true", "-DSWF_FAST=1"]


def build(force=False, verbose=False):
    if force or stale():
        _compile_link(OUT, NVCC_FLAGS, os.path.join(HERE, "..", "build", "obj"), verbose)
    if force or stale(OUT_FAST):
        _compile_link(OUT_FAST, FAST_FLAGS, os.path.join(HERE, "..", "build", "obj_fast"))
    build_host(force)
    return OUT


def build_variant(name, defines):
    """Developer A/B builds: paper_1705_00614_b200/variants/libswf_<name>.so with
    extra -D flags or raw nvcc flags (arguments starting with '-'); select one
    at run time with SWF_LIB=..."""
    vdir = os.path.join(HERE, "variants")
    os.makedirs(vdir, exist_ok=True)
    out = os.path.join(vdir, f"libswf_{name}.so")
    extra = [d if d.startswith("-") else f"-D{d}" for d in defines]
    _compile_link(out, NVCC_FLAGS + extra, os.path.join(HERE, "..", "build", "obj_" + name))
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "variant":  # build.py variant NAME [DEF=V ...]
        print(build_variant(sys.argv[2], sys.argv[3:]))
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(OUT)
