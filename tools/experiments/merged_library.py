"""Driver experiment: does one library holding every trace kernel of the
headline set restore faster than the 96 per-binary libraries?

    python tools/experiments/merged_library.py build DIR      # save + merged cubin
    python tools/experiments/merged_library.py time DIR split|merged   (fresh process each)

Timed per phase in a fresh context: cuLibraryLoadData of every cubin, the
first touch of each library's module (cuLibraryGetGlobal), cuLibraryGetKernel
of every entry, cuKernelGetFunction of every kernel (the lazy function load).
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
CUDA = "/usr/local/cuda/bin/"


def entries_ptx(images):
    out = [".version 8.8\n.target sm_100a\n.address_size 64\n\n",
           ".extern .func fdy_trace_body(.param .b64 a0, .param .b32 a1, .param .b64 a2, "
           ".param .b32 a3, .param .b32 a4, .param .b32 a5);\n"]
    names = []
    for ordinal, image in enumerate(images):
        for i, (name, (size, hidden)) in enumerate(image.items()):
            ename = "b%d_%s" % (ordinal, name)
            names.append(ename)
            h = "fdy_hidden_%d_%d" % (ordinal, i)
            if hidden:
                out.append(".global .align 4 .u32 %s[%d] = {%s};\n" % (h, len(hidden), ", ".join(map(str, hidden))))
            out.append(".visible .entry %s(\n\t.param .align 8 .b8 %s_param_0[%d]\n)\n{\n" % (ename, ename, size))
            out.append("\t.reg .b64 %rd<5>;\n\tmov.b64 %rd1, " + ename + "_param_0;\n\tcvta.param.u64 %rd2, %rd1;\n")
            out.append(("\tmov.u64 %%rd3, %s;\n\tcvta.global.u64 %%rd4, %%rd3;\n" % h) if hidden else "\tmov.u64 %rd4, 0;\n")
            out.append("\t{\n\t.param .b64 p0;\n\t.param .b32 p1;\n\t.param .b64 p2;\n\t.param .b32 p3;\n"
                       "\t.param .b32 p4;\n\t.param .b32 p5;\n")
            out.append("\tst.param.b64 [p0], %%rd2;\n\tst.param.b32 [p1], %d;\n\tst.param.b64 [p2], %%rd4;\n"
                       "\tst.param.b32 [p3], %d;\n\tst.param.b32 [p4], %d;\n\tst.param.b32 [p5], 0;\n"
                       % (size, len(hidden), (ordinal << 16) | i))
            out.append("\tcall.uni fdy_trace_body, (p0, p1, p2, p3, p4, p5);\n\t}\n\tret;\n}\n")
    return "".join(out), names


def build(d):
    import fndg
    import paper_2604_06664_b200 as foundry
    arch = os.path.join(d, "a")
    if not os.path.exists(os.path.join(arch, "manifest")):
        foundry.save(foundry.workload_from_text(open(foundry.workload_path("qwen3-235b-a22b")).read()), arch)
    bdir = os.path.join(arch, "binaries")
    bins = sorted(f for f in os.listdir(bdir) if f.endswith(".bin"))
    images = [fndg.kernel_image(open(os.path.join(bdir, f), "rb").read()) for f in bins]
    ptx, names = entries_ptx(images)
    open(os.path.join(d, "merged.ptx"), "w").write(ptx)
    body = os.path.join(ROOT, "paper_2604_06664_b200", "_build", "trace_body.ptx")
    t0 = time.time()
    subprocess.run([CUDA + "ptxas", "-arch=sm_100a", "-O3", "-c", body, "-o", os.path.join(d, "body.o")], check=True)
    subprocess.run([CUDA + "ptxas", "-arch=sm_100a", "-O3", "-c", os.path.join(d, "merged.ptx"), "-o",
                    os.path.join(d, "merged.o")], check=True)
    subprocess.run([CUDA + "nvlink", "-arch=sm_100a", os.path.join(d, "body.o"), os.path.join(d, "merged.o"), "-o",
                    os.path.join(d, "merged.cubin")], check=True)
    print(json.dumps({"entries": len(names), "compile_s": time.time() - t0,
                      "merged_bytes": os.path.getsize(os.path.join(d, "merged.cubin")),
                      "split_bytes": sum(os.path.getsize(os.path.join(bdir, f)) for f in os.listdir(bdir)
                                         if f.endswith(".cubin"))}))


def timed(d, mode):
    from cuda.bindings import driver as cu

    def ok(r):
        err = r[0] if isinstance(r, tuple) else r
        assert err == cu.CUresult.CUDA_SUCCESS, err
        return r[1] if isinstance(r, tuple) and len(r) == 2 else r

    t = {}
    s = time.perf_counter()
    ok(cu.cuInit(0))
    dev = ok(cu.cuDeviceGet(0))
    ctx = ok(cu.cuDevicePrimaryCtxRetain(dev))
    ok(cu.cuCtxSetCurrent(ctx))
    t["context_ms"] = (time.perf_counter() - s) * 1e3
    bdir = os.path.join(d, "a", "binaries")
    files = ([os.path.join(d, "merged.cubin")] if mode == "merged" else
             sorted(os.path.join(bdir, f) for f in os.listdir(bdir) if f.endswith(".cubin")))
    blobs = [open(f, "rb").read() for f in files]
    s = time.perf_counter()
    libs = [ok(cu.cuLibraryLoadData(b, None, None, 0, None, None, 0)) for b in blobs]
    t["library_load_ms"] = (time.perf_counter() - s) * 1e3
    s = time.perf_counter()
    for lib in libs:
        r = cu.cuLibraryGetGlobal(lib, b"fdy_trace_context")
        assert r[0] == cu.CUresult.CUDA_SUCCESS, r[0]
    t["first_touch_ms"] = (time.perf_counter() - s) * 1e3
    s = time.perf_counter()
    kernels = []
    for lib in libs:
        n = ok(cu.cuLibraryGetKernelCount(lib))
        ks = ok(cu.cuLibraryEnumerateKernels(n, lib))
        kernels.extend(ks)
    t["enumerate_ms"] = (time.perf_counter() - s) * 1e3
    s = time.perf_counter()
    for k in kernels:
        ok(cu.cuKernelGetFunction(k))
    t["function_load_ms"] = (time.perf_counter() - s) * 1e3
    t["kernels"] = len(kernels)
    t["libraries"] = len(libs)
    t["mode"] = mode
    print(json.dumps(t))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2])
    else:
        timed(sys.argv[2], sys.argv[3])
