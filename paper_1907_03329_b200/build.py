"""In-tree build of the CUDA engine (sm_100a) and the test oracles.

    python -m paper_1907_03329_b200.build      # or __graft_entry__.build()

Outputs (git-ignored, travel to the GPU box with the snapshot):
    paper_1907_03329_b200/libesrnn_b200.so     product: CUDA kernels + C-ABI
    oracle/liboracle_esrnn.so                  test oracle (plain C)
    oracle/_ref/libesrnn_ref.so                reference shim (only when /root/reference exists)
    build/cpp_api_test                         C++ drop-in API test driver (tests/cpp)
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_1907_03329_b200"
CSRC = PKG / "csrc"
INC = ROOT / "include"
BUILD = ROOT / "build"
LIB = PKG / "libesrnn_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-ffp-contract=off",
           "-I" + str(INC), "-I" + str(CSRC)]


def _run(cmd: list[str], cwd: Path | None = None) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=cwd)


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _torch_nccl_dir() -> str | None:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    if spec is None or not spec.submodule_search_locations:
        return None
    for base in spec.submodule_search_locations:
        d = Path(base) / "nccl" / "lib"
        if (d / "libnccl.so.2").exists():
            return str(d)
    return None


def build_engine(force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    deps = [*CSRC.glob("*.cu"), *CSRC.glob("*.cuh"), *CSRC.glob("*.h"), *CSRC.glob("*.cpp"), INC / "esrnn_b200.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    objs = []
    for src in sorted(CSRC.glob("*.cu")):
        obj = BUILD / (src.stem + ".o")
        _run([NVCC, *NVFLAGS, "-Xptxas", "-v", "-c", str(src), "-o", str(obj)])
        objs.append(str(obj))
    for src in sorted(CSRC.glob("*.cpp")):
        obj = BUILD / (src.stem + ".o")
        opt = "-O3" if src.stem in ("mt64", "ingest") else "-O2"
        _run(["g++", "-std=c++17", opt, "-fPIC", "-pthread", "-ffp-contract=off", "-I" + str(INC),
              "-I" + str(Path(NVCC).parent.parent / "include"), "-c", str(src), "-o", str(obj)])
        objs.append(str(obj))
    # Link the NCCL that torch bundles (2.28.x) so a process that also imports torch sees one
    # libnccl.so.2; fall back to the system copy (2.27.3) when the wheel is absent.
    nccl_dir = _torch_nccl_dir()
    link = ["-L" + nccl_dir, "-l:libnccl.so.2", "-Xlinker", "-rpath," + nccl_dir] if nccl_dir else \
        ["-L/usr/lib/x86_64-linux-gnu", "-lnccl"]
    _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *objs, "-Xlinker", "-Bsymbolic", *link])
    return LIB


def build_oracle() -> None:
    _run(["make", "-s", "all"], cwd=ROOT / "oracle")


def build_cpp_tests() -> None:
    src = ROOT / "tests" / "cpp" / "cpp_api_test.cpp"
    if not src.exists():
        return
    out = BUILD / "cpp_api_test"
    deps = [src, *(INC / "esrnn_b200").glob("*.hpp"), INC / "esrnn_b200.h"]
    if not _stale(out, deps) and not _stale(out, [LIB]):
        return
    BUILD.mkdir(exist_ok=True)
    _run(["g++", "-std=c++20", "-O2", "-I" + str(INC), str(src), "-o", str(out), "-L" + str(PKG), "-lesrnn_b200",
          "-Wl,-rpath,$ORIGIN/../paper_1907_03329_b200"])


REF_PROJ = Path("/root/reference/proj")


def _nlohmann_dir() -> str | None:
    """nlohmann/json 3.11.3 as vendored by cudnn_frontend in this image: the reference's
    checkpoint.hpp / commands.hpp / report.hpp include <json.hpp> from its (absent) vendor/."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    roots = [Path(sys.prefix) / "lib" / f"python{sys.version_info.major}.{sys.version_info.minor}" / "site-packages"]
    if spec and spec.submodule_search_locations:
        roots += [Path(b).parent for b in spec.submodule_search_locations]
    for r in roots:
        d = r / "include" / "cudnn_frontend" / "thirdparty" / "nlohmann"
        if (d / "json.hpp").exists():
            return str(d)
    return None


def build_reference_acceptance() -> None:
    """The reference's own acceptance suite (proj/tests/acceptance.cpp, criteria 1-9),
    compiled UNMODIFIED from /root/reference with only esrnn/trainer.hpp swapped for the
    drop-in (include overlay tests/cpp/overlay/esrnn/trainer.hpp): its Trainer calls,
    commands.hpp's cmd_train and checkpoint.hpp then run on the B200 engine.  Built here
    (the reference tree exists only in this container); the binary travels to the GPU box
    in build/.  Skipped when the reference tree or nlohmann/json is absent."""
    src = REF_PROJ / "tests" / "acceptance.cpp"
    js = _nlohmann_dir()
    if not src.exists() or js is None:
        print("reference acceptance: reference tree or nlohmann/json absent, keeping prebuilt build/ref_acceptance")
        return
    out = BUILD / "ref_acceptance"
    ov = ROOT / "tests" / "cpp" / "overlay"
    deps = [src, *(REF_PROJ / "include" / "esrnn").glob("*.hpp"), *(INC / "esrnn_b200").glob("*.hpp"),
            INC / "esrnn_b200.h", *ov.rglob("*.hpp")]
    if not _stale(out, deps) and not _stale(out, [LIB]):
        return
    BUILD.mkdir(exist_ok=True)
    _run(["g++", "-std=gnu++20", "-O2", "-I" + str(ov), "-I" + str(REF_PROJ / "include"), "-I" + str(INC),
          "-I" + js, str(src), "-o", str(out), "-L" + str(PKG), "-lesrnn_b200",
          "-Wl,-rpath,$ORIGIN/../paper_1907_03329_b200"])


def build_all(force: bool = False) -> None:
    build_engine(force)
    build_oracle()
    build_cpp_tests()
    build_reference_acceptance()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
