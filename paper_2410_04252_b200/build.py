"""In-tree build of the native pieces (no JIT cache, so the .so files travel
with the repo snapshot to the GPU box).

  libqrt.so          CUDA kernels + C ABI (include/qrt.h), sm_100a only
  libqrtile_b200.so  host C++ drop-in of the reference qrtile API, on libqrt
  _qrtile*.so        pybind11 module over libqrtile_b200 (tests, bench)

Run ``python -m paper_2410_04252_b200.build`` or call :func:`build`.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
BUILD = PKG / "_build"
SITE = Path(sysconfig.get_paths()["purelib"])
NCCL = SITE / "nvidia" / "nccl"
JSON_DIR = SITE / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SRCS = ["qrt_abi.cu", "qrt_gates.cu", "qrt_light.cu", "qrt_reorder.cu", "qrt_pauli.cu", "qrt_coset.cu"]
HOST_SRCS = ["qubit_core.cpp", "relayout.cpp", "tiling_qsu.cpp", "tiling_evc.cpp", "generators.cpp",
             "device_state.cpp"]

LIBQRT = PKG / "libqrt.so"
LIBQRT_CHECKED = PKG / "libqrt_checked.so"
BUILD_CHECKED = PKG / "_build_checked"
LIBHOST = PKG / "libqrtile_b200.so"
EXT = PKG / ("_qrtile" + sysconfig.get_config_var("EXT_SUFFIX"))


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str]) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("build step failed: " + " ".join(cmd[:3]) + " ...")


def _headers() -> list[Path]:
    return (list((PKG / "csrc").glob("*.h")) + [ROOT / "include" / "qrt.h"]
            + list((PKG / "host" / "include" / "qrtile").glob("*.hpp")))


def build_variant(name: str, defines: list[str]) -> Path:
    """An experiment build: libqrt_<name>.so from the same sources with extra
    -D defines, objects in _build_<name>.  Preload it (LD_PRELOAD) next to the
    product library for a same-box A/B of a compile-time alternative."""
    return build_libqrt(defines=defines, bdir=PKG / f"_build_{name}", out=PKG / f"libqrt_{name}.so")


def build_libqrt(checked: bool = False, defines: list[str] | None = None, bdir: Path | None = None,
                 out: Path | None = None) -> Path:
    """libqrt.so, or with checked=True libqrt_checked.so: the same kernels with
    -DQRT_CHECKS device-side bounds / pipeline checks (tests preload it)."""
    bdir = bdir or (BUILD_CHECKED if checked else BUILD)
    out = out or (LIBQRT_CHECKED if checked else LIBQRT)
    defines = list(defines or []) + (["QRT_CHECKS"] if checked else [])
    bdir.mkdir(exist_ok=True)
    objs, jobs = [], []
    for src in CU_SRCS:
        s = PKG / "csrc" / src
        o = bdir / (src + ".o")
        objs.append(o)
        if _stale(o, [s] + _headers()):
            jobs.append([NVCC, "-std=c++17", *ARCH, "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
                         *[f"-D{d}" for d in defines],
                         "-I", str(ROOT / "include"), "-I", str(NCCL / "include"),
                         "-c", str(s), "-o", str(o)])
    with ThreadPoolExecutor(max_workers=4) as ex:
        list(ex.map(_run, jobs))
    if _stale(out, objs):
        _run([NVCC, "-shared", *ARCH, "-o", str(out), *map(str, objs),
              "-L", str(NCCL / "lib"), "-l:libnccl.so.2",
              "-Xlinker", "-rpath," + str(NCCL / "lib")])
    return out


def build_host() -> Path:
    import pybind11

    BUILD.mkdir(exist_ok=True)
    inc = ["-I", str(PKG / "host" / "include"), "-I", str(ROOT / "include"), "-I", str(JSON_DIR)]
    flags = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra"]
    objs, jobs = [], []
    for src in HOST_SRCS:
        s = PKG / "host" / "src" / src
        o = BUILD / (src + ".o")
        objs.append(o)
        if _stale(o, [s] + _headers()):
            jobs.append(["g++", *flags, *inc, "-c", str(s), "-o", str(o)])
    with ThreadPoolExecutor(max_workers=8) as ex:
        list(ex.map(_run, jobs))
    if _stale(LIBHOST, objs + [LIBQRT]):
        _run(["g++", "-shared", "-o", str(LIBHOST), *map(str, objs), "-L", str(PKG), "-l:libqrt.so",
              "-Wl,-rpath,$ORIGIN", "-lpthread"])
    bind = PKG / "python" / "bindings.cpp"
    if _stale(EXT, [bind, LIBHOST] + _headers()):
        py_inc = sysconfig.get_paths()["include"]
        _run(["g++", *flags, "-Wno-unused-parameter", *inc, "-I", pybind11.get_include(), "-I", py_inc,
              "-shared", "-o", str(EXT), str(bind), "-L", str(PKG), "-l:libqrtile_b200.so", "-l:libqrt.so",
              "-Wl,-rpath,$ORIGIN"])
    return EXT


def build_oracle() -> None:
    """The checker: C restatement always, the real reference when its sources exist."""
    _run(["make", "-s", "-C", str(ROOT / "oracle"), "oracle"])
    if Path("/root/reference/proj/src").is_dir():
        _run(["make", "-s", "-j8", "-C", str(ROOT / "oracle"), "ref"])


def build() -> None:
    build_libqrt()
    build_host()
    build_libqrt(checked=True)
    build_oracle()


if __name__ == "__main__":
    build()
    print("built", LIBQRT.name, LIBHOST.name, EXT.name)
