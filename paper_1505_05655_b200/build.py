"""Build recipe for libgpcx.so (sm_100a) -- plain nvcc / g++, no torch JIT.

The shared library is built IN-TREE (paper_1505_05655_b200/lib/) so it
travels with the repo snapshot to the GPU box.  Objects are cached under
paper_1505_05655_b200/build/ and rebuilt when a source or header is newer.

    python -m paper_1505_05655_b200.build          # build if stale
    python -m paper_1505_05655_b200.build --force  # rebuild everything
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libgpcx.so"
SERVE_BIN = LIB_DIR / "gpcx-serve"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = ["lut.cu", "synth.cu", "sgemm.cu", "tc_gemm.cu", "demosaic.cu", "lsq.cu"]
CPP_SOURCES = [
    "status.cpp",
    "capi.cpp",
    "host/wire.cpp",
    "host/task_spec.cpp",
    "host/runtime.cpp",
    "host/executor.cpp",
    "host/peer.cpp",
    "host/devinfo.cpp",
    "host/registry.cpp",
    "host/tcp.cpp",
    "host/server.cpp",
]

NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "--expt-relaxed-constexpr", "-Xptxas", "-v", f"-I{ROOT / 'include'}",
]
CXX_FLAGS = [
    "-O2", "-g", "-std=c++20", "-fPIC", "-Wall", "-Wextra", "-pthread",
    f"-I{CUDA_HOME / 'include'}", f"-I{ROOT / 'include'}",
]


def _headers() -> list[Path]:
    return list(CSRC.rglob("*.hpp")) + list(CSRC.rglob("*.cuh")) + list((ROOT / "include").glob("*.h"))


def _stale(out: Path, src: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return src.stat().st_mtime > t or any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], log: Path | None = None) -> str:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
        raise RuntimeError(f"build step failed: {cmd[-1]}")
    out = proc.stdout + proc.stderr
    if log is not None:
        log.write_text(out)
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    deps = _headers()
    jobs = []
    objs = []
    for rel in CU_SOURCES:
        src = CSRC / rel
        obj = OBJ / (rel.replace("/", "_") + ".o")
        objs.append(obj)
        if force or _stale(obj, src, deps):
            jobs.append(([NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)], OBJ / (obj.name + ".ptxas.txt")))
    for rel in CPP_SOURCES:
        src = CSRC / rel
        obj = OBJ / (rel.replace("/", "_") + ".o")
        objs.append(obj)
        if force or _stale(obj, src, deps):
            jobs.append((["g++", *CXX_FLAGS, "-c", str(src), "-o", str(obj)], None))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            list(ex.map(lambda j: _run(*j), jobs))
    if force or jobs or not LIB.exists():
        _run([NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", str(LIB), *map(str, objs),
              "-Xlinker", f"-rpath,{CUDA_HOME / 'lib64'}", "-lpthread"])
    serve_src = CSRC / "tools" / "gpcx_serve.cpp"
    if serve_src.exists() and (force or _stale(SERVE_BIN, serve_src, deps + [LIB])):
        _run(["g++", *CXX_FLAGS, str(serve_src), "-o", str(SERVE_BIN), f"-L{LIB_DIR}", "-lgpcx",
              f"-Wl,-rpath,$ORIGIN", f"-Wl,-rpath,{CUDA_HOME / 'lib64'}",
              f"-L{CUDA_HOME / 'lib64'}", "-lcudart"])
    if verbose:
        print(f"built {LIB}")
    return LIB


TSAN_LIB = LIB_DIR / "tsan" / "libgpcx.so"


def build_tsan(verbose: bool = False) -> Path:
    """ThreadSanitizer build of the host side (server pipeline, runtime,
    registry, C ABI): the .cpp sources with -fsanitize=thread, linked with
    the regular CUDA objects into lib/tsan/libgpcx.so.  Load it with
    GPCX_LIB_PATH=<that file> and LD_PRELOAD=libtsan.so (tools/tsan_server.sh)."""
    build()
    out_dir = OBJ / "tsan"
    out_dir.mkdir(parents=True, exist_ok=True)
    TSAN_LIB.parent.mkdir(parents=True, exist_ok=True)
    flags = [f for f in CXX_FLAGS if f not in ("-O2",)] + ["-O1", "-fsanitize=thread"]
    jobs, objs = [], []
    for rel in CPP_SOURCES:
        obj = out_dir / (rel.replace("/", "_") + ".o")
        objs.append(obj)
        jobs.append((["g++", *flags, "-c", str(CSRC / rel), "-o", str(obj)], None))
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(lambda j: _run(*j), jobs))
    cu_objs = [OBJ / (rel.replace("/", "_") + ".o") for rel in CU_SOURCES]
    _run(["g++", "-shared", "-fsanitize=thread", "-o", str(TSAN_LIB), *map(str, objs),
          *map(str, cu_objs), f"-L{CUDA_HOME / 'lib64'}", "-lcudart", "-lpthread",
          f"-Wl,-rpath,{CUDA_HOME / 'lib64'}"])
    if verbose:
        print(f"built {TSAN_LIB}")
    return TSAN_LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--tsan", action="store_true", help="also build lib/tsan/libgpcx.so")
    args = ap.parse_args()
    build(force=args.force, verbose=True)
    if args.tsan:
        build_tsan(verbose=True)


if __name__ == "__main__":
    main()
