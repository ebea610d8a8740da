"""First-light GPU check: fused materialize kernel + GPU CRC vs the C oracle.

Generates archives with the reference (oracle/_ref/ref_tool, test infra),
packs them with fdy_tool, runs the kernel through the C-ABI and compares the
re-encoded FNDG container byte for byte with oracle/foundry_oracle.c.
"""
import ctypes, json, os, subprocess, sys, tempfile, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle/_ref/ref_tool")
TOOL = os.path.join(ROOT, "paper_2604_06664_b200/fdy_tool")
lib = ctypes.CDLL(os.path.join(ROOT, "oracle/_build/liboracle.so"))
lib.fo_crc64.restype = ctypes.c_uint64
lib.fo_crc64.argtypes = [ctypes.c_char_p, ctypes.c_size_t]

def oracle(arch, rank, world, delta):
    m = json.load(open(arch + "/manifest"))
    g = open(arch + "/graphs.bin", "rb").read(); p = open(arch + "/patch.bin", "rb").read()
    out = ctypes.POINTER(ctypes.c_uint8)(); n = ctypes.c_size_t(); nr = ctypes.c_uint64()
    err = ctypes.create_string_buffer(512)
    base = m["allocator"]["base"]; fo = m["allocator"]["final_offset"]
    rc = lib.fo_materialize_container(g, len(g), p, len(p), ctypes.c_uint64(m["comm"]["real_binary_hash"]),
        rank, world, ctypes.c_uint64(base), ctypes.c_uint64(fo), ctypes.c_uint64(base + delta if delta else base),
        8, ctypes.byref(out), ctypes.byref(n), ctypes.byref(nr), err, 512)
    if rc: raise RuntimeError(err.value)
    b = ctypes.string_at(out, n.value); lib.fo_free(out); return b, m

work = tempfile.mkdtemp(prefix="fdy_qc_")
specs = {"micro": "micro", "moe": "moe-spmd",
         "llama3-8b": os.path.join(ROOT, "paper_2604_06664_b200/workloads/llama3-8b.spec"),
         "qwen3-235b": os.path.join(ROOT, "paper_2604_06664_b200/workloads/qwen3-235b-a22b.spec")}
ok = True
for name, spec in specs.items():
    arch = os.path.join(work, name)
    subprocess.run([REF, "save", spec, arch], check=True, capture_output=True)
    subprocess.run([TOOL, "pack", arch], check=True, capture_output=True)
    cases = [(0, 1, 0), (0, 1, 0x10000), (3, 8, 0x10000000000), (1, 4, 0x123450000)]
    for rank, world, delta in cases:
        exp, m = oracle(arch, rank, world, delta)
        nb = "0" if not delta else "%x" % (m["allocator"]["base"] + delta)
        out = os.path.join(work, "gpu.fndg")
        r = subprocess.run([TOOL, "gpu-materialize", arch, str(rank), str(world), nb, out, "20"],
                           capture_output=True, text=True)
        if r.returncode:
            print("FAIL run", name, rank, world, hex(delta), r.stderr); ok = False; continue
        got = open(out, "rb").read()
        same = got == exp
        ok &= same
        print(name, rank, world, hex(delta), "bit-exact" if same else "MISMATCH", r.stdout.strip())
    files = sorted(m["files"])
    r = subprocess.run([TOOL, "gpu-crc"] + [os.path.join(arch, f) for f in files], capture_output=True, text=True)
    for line, f in zip(r.stdout.splitlines(), files):
        d = open(os.path.join(arch, f), "rb").read()
        cpu = lib.fo_crc64(d, len(d))
        same = int(line.split()[0], 16) == cpu == m["files"][f]
        ok &= same
        if not same: print("CRC MISMATCH", name, f, line)
    print(name, "gpu crc", r.returncode, r.stderr.strip())
print("ALL OK" if ok else "FAILURES")
sys.exit(0 if ok else 1)
