"""In-tree build of the native library (no setuptools, no JIT cache).

    python -m paper_1704_08657_b200.build [--jobs N] [--force]

1. compiles the plan generator (host algebra + csrc/tools/gen_plans.cpp) and
   regenerates csrc/generated/ (files rewritten only when their text changes)
2. compiles host C++ with g++ and every .cu with nvcc for sm_100a
   (-gencode arch=compute_100a,code=sm_100a -lineinfo), in parallel
3. links paper_1704_08657_b200/lib/libdwt2d_b200.so (static cudart) and the
   C++ API test driver build/test_cpp_api
Incremental: an object is rebuilt when its source or any header is newer.
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = ROOT / "build"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libdwt2d_b200.so"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", shutil.which("g++") or "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-std=c++20", "-lineinfo", "--expt-relaxed-constexpr",
                  "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
                  "-Xptxas", "-v", f"-I{INCLUDE}"]
# host C++ keeps default visibility: the C++ API (include/dwt2d_b200/*.hpp)
# is exported next to the C ABI
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", f"-I{INCLUDE}", "-I/usr/local/cuda/include"]

HOST_SRCS = ["host/algebra.cpp", "host/wavelets.cpp", "host/schemes.cpp", "host/lowering.cpp", "host/io.cpp"]
RUNTIME_SRCS = ["runtime/capi.cpp"]


def _headers() -> list[Path]:
    hs = list(INCLUDE.rglob("*.h")) + list(INCLUDE.rglob("*.hpp"))
    hs += list(CSRC.rglob("*.cuh")) + list(CSRC.rglob("*.hpp"))
    return hs


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], log: Path | None = None) -> str:
    r = subprocess.run(cmd, capture_output=True, text=True)
    out = r.stdout + r.stderr
    if log is not None:
        log.write_text(" ".join(cmd) + "\n" + out)
    if r.returncode != 0:
        raise RuntimeError(f"command failed ({r.returncode}): {' '.join(cmd)}\n{out[-6000:]}")
    return out


def generate(force: bool = False) -> None:
    gen_bin = BUILD / "gen_plans"
    srcs = [CSRC / s for s in HOST_SRCS] + [CSRC / "tools/gen_plans.cpp"]
    hdrs = list(INCLUDE.rglob("*.hpp"))
    if force or _stale(gen_bin, srcs + hdrs):
        _run([CXX, "-std=c++20", "-O2", f"-I{INCLUDE}", *map(str, srcs), "-o", str(gen_bin)])
    tmp = BUILD / "gen_tmp"
    if tmp.exists():
        shutil.rmtree(tmp)
    tmp.mkdir(parents=True)
    _run([str(gen_bin), str(tmp)])
    outdir = CSRC / "generated"
    outdir.mkdir(exist_ok=True)
    fresh = {p.name for p in tmp.iterdir()}
    for p in tmp.iterdir():
        dst = outdir / p.name
        if not dst.exists() or dst.read_text() != p.read_text():
            shutil.copyfile(p, dst)
    for p in outdir.iterdir():
        if p.name not in fresh:
            p.unlink()
    shutil.rmtree(tmp)


def build(jobs: int | None = None, force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    (BUILD / "logs").mkdir(exist_ok=True)
    LIBDIR.mkdir(exist_ok=True)
    generate(force)
    hdrs = _headers()
    units = []  # (compiler, src, obj)
    for s in HOST_SRCS:
        units.append(("cxx", CSRC / s))
    for s in RUNTIME_SRCS:
        units.append(("cxx", CSRC / s))
    units.append(("nvcc", CSRC / "kernels/generic_step.cu"))
    units.append(("nvcc", CSRC / "kernels/exchange.cu"))
    for cu in sorted((CSRC / "generated").glob("*.cu")):
        units.append(("nvcc", cu))
    objs = []

    def compile_one(kind, src):
        obj = BUILD / "obj" / (src.relative_to(CSRC).as_posix().replace("/", "__") + ".o")
        obj.parent.mkdir(parents=True, exist_ok=True)
        if force or _stale(obj, [src] + hdrs):
            log = BUILD / "logs" / (obj.name + ".log")
            if kind == "cxx":
                _run([CXX, *CXXFLAGS, "-c", str(src), "-o", str(obj)], log)
            else:
                _run([NVCC, *NVFLAGS, "-c", str(src), "-o", str(obj)], log)
            if verbose:
                print("built", obj.name, flush=True)
        return obj

    with ThreadPoolExecutor(max_workers=jobs or max(2, os.cpu_count() or 2)) as ex:
        futs = [ex.submit(compile_one, k, s) for k, s in units]
        objs = [f.result() for f in futs]
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs),
              "-Xlinker", "-Bsymbolic", "-Xlinker", "--exclude-libs,ALL"], BUILD / "logs" / "link.log")
    cli_src = CSRC / "tools" / "dwt2d_cli.cpp"
    cli_bin = PKG / "bin" / "dwt2d"
    if force or _stale(cli_bin, [cli_src, LIB] + hdrs):
        cli_bin.parent.mkdir(exist_ok=True)
        _run([CXX, "-std=c++20", "-O2", f"-I{INCLUDE}", str(cli_src), "-o", str(cli_bin), f"-L{LIBDIR}",
              "-ldwt2d_b200", "-Wl,-rpath,$ORIGIN/../lib"], BUILD / "logs" / "dwt2d_cli.log")
    test_src = ROOT / "tests" / "cpp" / "test_cpp_api.cpp"
    test_bin = BUILD / "test_cpp_api"
    if test_src.exists() and (force or _stale(test_bin, [test_src, LIB] + hdrs)):
        _run([CXX, "-std=c++20", "-O2", f"-I{INCLUDE}", str(test_src), "-o", str(test_bin),
              f"-L{LIBDIR}", "-ldwt2d_b200", "-Wl,-rpath,$ORIGIN/../paper_1704_08657_b200/lib"], BUILD / "logs" / "test_cpp_api.log")
    return LIB


def build_oracle() -> bool:
    """Compile the reference oracle (test infrastructure) when the reference
    sources are present; on the GPU box only the prebuilt oracle/_ref files
    exist and this is a no-op."""
    if not Path("/root/reference/proj/src").exists():
        return False
    _run(["make", "-s", "-C", str(ROOT / "oracle")])
    return True


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--no-oracle", action="store_true")
    a = ap.parse_args(argv)
    lib = build(a.jobs, a.force, verbose=True)
    print("library:", lib)
    if not a.no_oracle:
        print("oracle built:", build_oracle())


if __name__ == "__main__":
    sys.exit(main())
