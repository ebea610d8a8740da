"""In-tree build of the native pieces (ninja, incremental).

Products (all inside the package directory so they travel with the repo
snapshot to the GPU box and are what the tests/bench load):

  libfoundry_b200.so          host runtime + sm_100a kernels + the C-ABI
                              (include/foundry_b200.h)
  _foundry<EXT>               pybind11 module mirroring the reference bindings
  trace_body.ptx              device body of the generated trace kernels
  fdy_tool                    CLI: save / pack / load / bench helpers
  foundry                     the reference's CLI (save/load/inspect/diff/bench)

Kernels compile with -gencode arch=compute_100a,code=sm_100a -lineinfo; there
is no other architecture and no JIT fallback.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"

CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NLOHMANN = Path(
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
)
ARCH = "-gencode arch=compute_100a,code=sm_100a"

HOST_SRCS = [
    "host/support.cpp",
    "host/graph_model.cpp",
    "host/archive.cpp",
    "host/template_store.cpp",
    "host/device_pack.cpp",
    "host/device.cpp",
    "host/workload.cpp",
    "host/save.cpp",
    "host/trace_module.cpp",
    "host/driver_api.cpp",
    "host/gpu_context.cpp",
    "host/staging.cpp",
    "host/capture.cpp",
    "host/pipeline.cpp",
    "host/tooling.cpp",
    "capi/capi_misc.cpp",
    "capi/capi_kernels.cpp",
    "capi/capi_session.cpp",
]
CU_SRCS = ["kernels/materialize.cu", "kernels/crc64.cu", "kernels/pack.cu", "kernels/fanout.cu"]
RDC_SRCS = ["kernels/serve.cu"]  # device runtime (graph device updates): -rdc + device link


def _ninja_bin() -> str:
    for cand in (shutil.which("ninja"), "/opt/prime-rl/.venv/bin/ninja"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("ninja not found")


def _write_ninja() -> Path:
    import pybind11

    py_inc = sysconfig.get_paths()["include"]
    ext = sysconfig.get_config_var("EXT_SUFFIX")
    inc = f"-I{CSRC}/include -I{ROOT}/include -I{CUDA}/include -I{NLOHMANN}"
    cxxflags = f"-std=c++20 -O2 -g -fPIC -Wall -Wextra -Wno-missing-field-initializers {inc}"
    nvflags = (
        f"-std=c++17 {ARCH} -O3 -lineinfo -Xcompiler -fPIC -Xptxas -v {inc} "
        "--expt-relaxed-constexpr"
    )
    cudart = CUDA / "lib64" / "libcudart_static.a"
    lines = [
        f"cxx = g++",
        f"nvcc = {CUDA}/bin/nvcc",
        f"cxxflags = {cxxflags}",
        f"nvflags = {nvflags}",
        "rule cxx",
        "  command = $cxx $cxxflags -MMD -MF $out.d -c $in -o $out",
        "  depfile = $out.d",
        "  deps = gcc",
        "  description = CXX $in",
        "rule nvcc",
        "  command = $nvcc $nvflags -MD -MF $out.d -c $in -o $out 2> $out.ptxas.log || "
        "(cat $out.ptxas.log; false)",
        "  depfile = $out.d",
        "  deps = gcc",
        "  description = NVCC $in",
        "rule nvcc_rdc",
        "  command = $nvcc $nvflags -rdc=true -MD -MF $out.d -c $in -o $out 2> $out.ptxas.log || "
        "(cat $out.ptxas.log; false)",
        "  depfile = $out.d",
        "  deps = gcc",
        "  description = NVCC-RDC $in",
        "rule dlink",
        f"  command = $nvcc {ARCH} -Xcompiler -fPIC -dlink $in -L{CUDA}/lib64 -lcudadevrt -o $out",
        "  description = DLINK $out",
        # no -lineinfo: the PTX is embedded into SAVE output, which must not depend on paths
        "rule ptx",
        f"  command = $nvcc -std=c++17 -arch=sm_100a -rdc=true -ptx -O3 -I{CSRC}/include $in -o $out",
        "  description = PTX $in",
        "rule embed",
        f"  command = {sys.executable} {CSRC}/tools/embed_ptx.py $in $out",
        "  description = EMBED $in",
        # -Bsymbolic: the library's own C++ symbols (namespace foundry, the
        # reference's names) bind inside it, so a process that also links the
        # reference cannot interpose them
        "rule link",
        f"  command = $cxx -shared -o $out $in {cudart} {CUDA}/lib64/libcudadevrt.a -ldl -lrt -lpthread "
        "-Wl,-soname,libfoundry_b200.so -Wl,-Bsymbolic",
        "  description = LINK $out",
        "rule pymod",
        f"  command = $cxx $cxxflags -shared -I{py_inc} -I{pybind11.get_include()} $in "
        f"-L{PKG} -lfoundry_b200 -Wl,-rpath,'$$ORIGIN' -o $out",
        "  description = PYMOD $out",
        "rule exe",
        f"  command = $cxx $cxxflags -rdynamic $in -L{PKG} -lfoundry_b200 -Wl,-rpath,'$$ORIGIN' -o $out",
        "  description = EXE $out",
    ]
    objs = []
    for src in HOST_SRCS:
        obj = BUILD / (src.replace("/", "_") + ".o")
        lines.append(f"build {obj}: cxx {CSRC / src}")
        objs.append(str(obj))
    for src in CU_SRCS:
        obj = BUILD / (src.replace("/", "_") + ".o")
        lines.append(f"build {obj}: nvcc {CSRC / src}")
        objs.append(str(obj))
    rdc_objs = []
    for src in RDC_SRCS:
        obj = BUILD / (src.replace("/", "_") + ".o")
        lines.append(f"build {obj}: nvcc_rdc {CSRC / src}")
        rdc_objs.append(str(obj))
    dl = BUILD / "device_link.o"
    lines.append(f"build {dl}: dlink {' '.join(rdc_objs)}")
    objs += rdc_objs + [str(dl)]
    ptx = BUILD / "trace_body.ptx"
    lines.append(f"build {ptx}: ptx {CSRC / 'kernels/trace_body.cu'}")
    lines.append(f"build {BUILD / 'trace_body_ptx.cpp'}: embed {ptx}")
    lines.append(f"build {BUILD / 'trace_body_ptx.o'}: cxx {BUILD / 'trace_body_ptx.cpp'}")
    objs.append(str(BUILD / "trace_body_ptx.o"))
    lib = PKG / "libfoundry_b200.so"
    lines.append(f"build {lib}: link {' '.join(objs)}")
    lines.append(f"build {PKG / 'fdy_tool'}: exe {CSRC / 'tools/fdy_tool.cpp'} | {lib}")
    lines.append(f"build {PKG / 'foundry'}: exe {CSRC / 'tools/foundry_cli.cpp'} | {lib}")
    lines.append(f"build {PKG / ('_foundry' + ext)}: pymod {CSRC / 'bindings/module.cpp'} | {lib}")
    BUILD.mkdir(parents=True, exist_ok=True)
    path = BUILD / "build.ninja"
    # in-tree paths relative to the build directory (ninja runs there): the
    # same build.ninja, depfiles and PTX `.file` lines wherever the tree is
    # checked out (the GPU box copies it to a scratch path), so a snapshot's
    # up-to-date objects are not rebuilt and SAVE's cubins stay byte-identical
    text = ("\n".join(lines) + "\n").replace(str(ROOT), os.path.relpath(ROOT, BUILD))
    if not path.exists() or path.read_text() != text:
        path.write_text(text)
    return path


def build(verbose: bool = False, jobs: int | None = None) -> None:
    ninja = _write_ninja()
    cmd = [_ninja_bin(), "-f", str(ninja)]
    if jobs:
        cmd += ["-j", str(jobs)]
    if verbose:
        cmd.append("-v")
    proc = subprocess.run(cmd, cwd=BUILD, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout[-20000:] + proc.stderr[-20000:])
        raise RuntimeError("native build failed")
    if verbose:
        sys.stdout.write(proc.stdout)


if __name__ == "__main__":
    build(verbose="-v" in sys.argv)
