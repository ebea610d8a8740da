#!/usr/bin/env python3
"""Benchmark: graph-set materialization on B200 (Foundry LOAD path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload qwen3-235b-a22b]

One "step" = one graph-set materialization for one rank: every member graph
of the archive (512 batch sizes, 1036 nodes each for the headline
Qwen3-235B-A22B-shaped TP8 set) expanded from the HBM-resident template store
by the fused K2 (diff) + K1 (relocation) + K3 (rank patch) kernel. Each process
is one GPU and one TP rank (rank = global rank % 8 of world 8), so per-GPU work
is fixed as N grows ("weak" scaling); there is no data-path collective.

JSON keys beyond the base contract:
  e2e          the same materialization through the C-ABI with host buffers
               (fdy_prepare_archive): archive files -> integrity (GPU CRC of the
               store, host CRC of the rest) -> fused kernel -> every member's
               parameters in host memory. The reference arm's e2e is its CPU
               path for the same work (verify_archive_integrity + PrepareFn).
  e2e_plain    the same call on the archive as the reference writes it (no
               templates.fdt): the template store is packed on the GPU first.
  e2e_servable LOAD to every graph servable (foundry.load): + cuLibraryLoadData,
               function loads, template graphs built + instantiated, with the
               driver-bound part broken out; next to the reference's load().
  roofline     HBM roofline of the fused kernel (algorithmic bytes / event time).
  cpu_baseline the reference's own CPU path (oracle/_ref) on this host's cores.
"""
from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
TP_WORLD = 8  # the headline set is TP8: every GPU materializes one rank's graph set


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", default="qwen3-235b-a22b")
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--load-steps", type=int, default=3)
    p.add_argument("--skip-load", action="store_true", help="skip the full-LOAD section (profiling)")
    p.add_argument("--fanout", choices=["host", "ipc", "chain"], default="ipc",
                   help="N>1: how the store reaches every GPU (ipc = GPU0 -> peers over NVLink)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--skip-tier-s", action="store_true", help="skip the model-shaped arena measurement")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def prepare_archives(workload: str, local_rank: int, barrier) -> tuple[str, str]:
    """Writes (once per node: local rank 0, into the node-local temp dir) the
    B200 archive and a reference-layout archive (no B200 artefacts) of the same
    spec with this build's SAVE, which is byte-identical to the reference's
    (tests/test_save.py). Every rank waits at `barrier` for its node's writer."""
    import paper_2604_06664_b200 as foundry

    root = os.path.join(tempfile.gettempdir(), "foundry_bench_" + workload)
    ours, plain = os.path.join(root, "b200"), os.path.join(root, "plain")
    done = os.path.join(root, "READY")
    # the cache is only reused by the exact build + spec that wrote it
    stamp = hashlib.sha1(open(foundry._foundry.__file__, "rb").read()
                         + open(foundry.workload_path(workload), "rb").read()).hexdigest()
    fresh = os.path.exists(done) and open(done).read() == stamp
    # The reference-layout archive carries the catalog's FNDB images but no
    # sm_100a cubins; LOAD turns each into a trace module (the emulation of
    # that binary on this GPU: ptxas + nvlink). The content-addressed cache the
    # B200 SAVE filled makes that a lookup on every rank and every run, so
    # the reference-written LOAD is timed without the emulation's compile.
    os.environ.setdefault("FOUNDRY_CUBIN_CACHE", os.path.join(root, "cubin_cache"))
    if local_rank == 0 and not fresh:
        shutil.rmtree(root, ignore_errors=True)
        os.makedirs(root)
        spec = foundry.workload_from_text(open(foundry.workload_path(workload)).read())
        foundry.save(spec, ours)
        foundry.save(spec, plain, b200_artifacts=False)
        open(done, "w").write(stamp)
    barrier()
    return ours, plain


def tier_s_archive(archive: str) -> str:
    """The headline archive with model-shaped argument blocks (SURVEY §8(d) tier
    S: every third kernel node a 1720-byte GEMM-like block with embedded device
    pointers, ragged tails, member-varying grids; tests/tier_s.py), packed.
    Cached next to the archive it is derived from."""
    import paper_2604_06664_b200 as foundry
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import tier_s

    out = os.path.join(os.path.dirname(archive), "tier_s")
    done = os.path.join(os.path.dirname(archive), "TIER_S_READY")
    if not os.path.exists(done):
        shutil.rmtree(out, ignore_errors=True)
        tier_s.make_tier_s(archive, out, foundry._foundry._crc64)
        foundry._foundry._pack_store(out)
        open(done, "w").write("ok")
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + q, "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [int(r[0]) for r in self.rows if r[0].isdigit()]
        busy = [int(r[0]) for r in self.rows if r[0].isdigit() and r[6].isdigit() and int(r[6]) > 0]
        reasons = set()
        for r in self.rows:
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"], r[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(busy or sm), "sm_max_mhz": int(self.rows[0][1]),
                "samples": len(self.rows), "samples_busy": len(busy), "reasons": sorted(reasons)}


def reference_load_ms(archive: str, rank: int, world: int, lanes: int, reps: int) -> dict | None:
    if not os.path.exists(REF_TOOL):
        return None
    r = subprocess.run([REF_TOOL, "time-load", archive, str(rank), str(world), str(lanes), str(reps)],
                       capture_output=True, text=True)
    return json.loads(r.stdout) if r.returncode == 0 else None


def reference_materialize_ms(archive: str, rank: int, world: int, lanes: int, reps: int,
                             warmup: int = 1) -> dict | None:
    if not os.path.exists(REF_TOOL):
        return None
    r = subprocess.run([REF_TOOL, "time-materialize", archive, str(rank), str(world), str(lanes),
                        str(reps), str(warmup)], capture_output=True, text=True)
    return json.loads(r.stdout) if r.returncode == 0 else None


def oracle_port_ms(archive: str, rank: int, world: int, lanes: int, reps: int) -> dict:
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle

    orc = Oracle(os.path.join(ROOT, "oracle", "_build", "liboracle.so"))
    times = []
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        orc.materialize_archive(archive, rank, world, 0x10000, lanes)
        times.append((time.perf_counter() - t0) * 1e3)
    return {"best_ms": min(times[1:]), "mean_ms": statistics.mean(times[1:]), "reps": reps,
            "lanes": lanes}


def spec_path(workload: str) -> str:
    """The bundled tier-R spec, resolved by path (the reference arm must not
    import this build's package)."""
    return os.path.join(ROOT, "paper_2604_06664_b200", "workloads", workload + ".spec")


def reference_archive(workload: str) -> str | None:
    """The workload's archive written by the reference itself (ref_tool save,
    foundry::save pipeline.cpp:249-405), so the reference arm runs none of
    this build's code. Byte-identical to this build's SAVE (tests/test_save.py)."""
    if not os.path.exists(REF_TOOL):
        return None
    spec = spec_path(workload)
    root = os.path.join(tempfile.gettempdir(), "foundry_refarm_" + workload)
    stamp = hashlib.sha1(open(REF_TOOL, "rb").read() + open(spec, "rb").read()).hexdigest()
    done = os.path.join(root, "READY")
    out = os.path.join(root, "archive")
    if not (os.path.exists(done) and open(done).read() == stamp):
        shutil.rmtree(root, ignore_errors=True)
        os.makedirs(root)
        r = subprocess.run([REF_TOOL, "save", spec, out], capture_output=True, text=True)
        if r.returncode != 0:
            return None
        open(done, "w").write(stamp)
    return out


def graph_counts(archive: str) -> tuple[int, int, int]:
    """(graphs, templates, nodes) of an archive from its manifest and the FNDG
    locator table of graphs.bin (graph_model.cpp:244-293) — plain file reads,
    identical for both arms."""
    import struct

    with open(os.path.join(archive, "manifest")) as f:
        grouping = json.load(f)["grouping"]
    nodes = 0
    with open(os.path.join(archive, "graphs.bin"), "rb") as f:
        head = f.read(10)
        (count,) = struct.unpack_from("<I", head, 6)
        locs = f.read(28 * count)
        for i in range(count):
            (off,) = struct.unpack_from("<Q", locs, 28 * i + 4)
            f.seek(off + 4)
            nodes += struct.unpack("<I", f.read(4))[0]
    return grouping["total"], grouping["templates"], nodes


def bench_config(workload: str, archive: str, wrank: int) -> dict:
    """The `config` both arms print (the driver compares them for equality)."""
    graphs, templates, nodes = graph_counts(archive)
    return {"workload": workload + "~ tier-R decode graph set, TP8: rank %d of 8 per GPU" % wrank,
            "graphs": graphs, "templates": templates, "nodes": nodes, "rank": wrank, "world": TP_WORLD,
            "parallelism": "replicas (one TP rank per GPU)",
            "value": "graph-set materialization with the template store resident in HBM (ours) / "
                     "the reference CPU path (reference)",
            "e2e": "archive files -> integrity -> every member graph's parameters in host memory",
            "l2": "flushed between timed device steps (256 MiB memset + 256 MiB read of unrelated "
                  "buffers, outside the events)"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_serve_ms(archive: str, rank: int, world: int, lanes: int, reps: int) -> dict | None:
    if not os.path.exists(REF_TOOL):
        return None
    r = subprocess.run([REF_TOOL, "time-serve", archive, str(rank), str(world), str(lanes), str(reps)],
                       capture_output=True, text=True)
    return json.loads(r.stdout) if r.returncode == 0 else None


def cold_process_load(args, local: int, samples: int = 5) -> dict:
    """Wall clock of a fresh process from exec to every template servable:
    `foundry load --archive <headline> --rank 0 --world 8` (CUDA context
    creation + LOAD, stamped when the CLI's flushed "ready" line arrives),
    per-template execs and share_execs, next to a fresh process that only
    creates the CUDA context (`fdy_tool cuda-init`, stamped at its own 'ready'
    line once the context exists, like the LOAD processes). The three kinds run
    interleaved, `samples` rounds in a rotating order with a 1 s settle before
    each process, so drift of the box and the previous process's teardown hit
    all of them alike; median and range per kind. `device_open_ms` / `load_ms` split the LOAD
    process at its device-open stamp (FOUNDRY_DEBUG timeline); the CLI asks
    the kernel to read the archive ahead (posix_fadvise) before it creates
    the context. `process_exit` adds the teardown (graphs, libraries, context)."""
    archive, _ = prepare_archives(args.workload, 0, lambda: None)
    pkg = os.path.join(ROOT, "paper_2604_06664_b200")
    runs = {"cuda_init": [os.path.join(pkg, "fdy_tool"), "cuda-init", str(local)]}
    base = [os.path.join(pkg, "foundry"), "load", "--archive", archive, "--rank", "0", "--world",
            str(TP_WORLD), "--device", str(local)]
    runs["share_execs"] = base + ["--share-execs"]
    runs["per_template"] = base
    # one untimed fresh process first: the box's very first context creation after
    # idle (driver / GPU wake-up) is not part of any load
    subprocess.run(runs["cuda_init"], capture_output=True)
    walls = {k: [] for k in runs}
    exits = {k: [] for k in runs}
    opens = {k: [] for k in runs}
    env = dict(os.environ, FOUNDRY_DEBUG="1")
    names = list(runs)
    for r in range(samples):
        # rotate the order each round and let the driver finish tearing down
        # the previous process first: a context created right after a heavy
        # process exits is slower, whichever kind it belongs to
        for name in names[r % len(names):] + names[:r % len(names)]:
            cmd = runs[name]
            time.sleep(1.0)
            t0 = time.perf_counter()
            p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, env=env)
            t_ready = None
            for line in p.stdout:  # the CLI flushes its "ready" line when LOAD returns
                if t_ready is None and " ready: " in line:
                    t_ready = time.perf_counter()
            err = p.stderr.read()
            rc = p.wait()
            t_exit = time.perf_counter()
            if rc != 0:
                continue
            walls[name].append(((t_ready or t_exit) - t0) * 1e3)
            exits[name].append((t_exit - t0) * 1e3)
            for line in err.splitlines():  # "[foundry]   812.3 ms  device open"
                if line.endswith("  device open"):
                    opens[name].append(float(line.split()[1]))

    def stat(xs):
        return None if not xs else {"median": statistics.median(xs), "min": min(xs), "max": max(xs), "n": len(xs)}

    out = {k: stat(v) for k, v in walls.items()}
    out["process_exit"] = {k: stat(v) for k, v in exits.items()}
    out["device_open_ms"] = {k: stat(v) for k, v in opens.items() if v}
    out["load_ms"] = {k: stat([w - o for w, o in zip(walls[k], opens[k])]) for k in runs if opens[k]}
    return out


def full_load_stats(foundry, archive, wrank, lanes, steps, barrier, reduce_max, **kw) -> dict:
    """LOAD to every graph servable through the public API (foundry.load):
    archive files -> integrity -> catalog restore (cuLibraryLoadData) ->
    fused materialization -> template graphs built + instantiated (and, with
    share_execs, every other template's functions loaded) -> member parameters
    resident in HBM, representatives on the host. One warm-up, then `steps`
    LOADs; per-phase breakdown averaged, wall as median/min/max (max over
    ranks of the median)."""
    h = foundry.load(archive, rank=wrank, world=TP_WORLD, prepare_lanes=lanes, **kw)  # warm-up
    h.close()
    walls, bds = [], []
    for _ in range(steps):
        barrier()
        t0 = time.perf_counter()
        h = foundry.load(archive, rank=wrank, world=TP_WORLD, prepare_lanes=lanes, **kw)
        walls.append((time.perf_counter() - t0) * 1e3)
        bds.append(dict(h.timings(), instantiate_calls=h.counters()["exec.instantiate_calls"]))
        h.close()
    bd = {k: statistics.mean(b[k] for b in bds) for k in bds[0]}
    driver = sum(bd.get(k, 0) for k in ("restore_ms", "build_ms", "instantiate_ms", "function_load_ms"))
    return {"value": reduce_max(statistics.median(walls)), "unit": "ms", "min": min(walls), "max": max(walls),
            "steps": steps, "instantiate_calls": bd["instantiate_calls"],
            "driver_bound_ms": driver,
            "h2d_bytes_per_step": int(bd.get("h2d_bytes", 0)), "d2h_bytes_per_step": int(bd.get("d2h_bytes", 0)),
            "breakdown": {k: v for k, v in bd.items() if k.endswith("_ms") and k != "crc_kernel_ms"}}


def run_reference(args, grank, gworld):
    """--impl reference: the reference's own CPU implementation of the path on
    this host's cores (oracle/_ref/ref_tool over the unmodified reference), on
    an archive the reference's own save wrote. Imports nothing from this
    build. value = e2e = verify_archive_integrity + PrepareFn of every member
    on all host threads; the full load() and serve+replay sweep ride along."""
    if grank != 0:
        return
    lanes = os.cpu_count() or 1
    plain = reference_archive(args.workload)
    if plain is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_tool is not built "
                          "(make -C oracle ref needs /root/reference)"}), flush=True)
        return
    wrank = 0
    res = reference_materialize_ms(plain, wrank, TP_WORLD, lanes, args.steps, args.warmup)
    kind = "reference"
    if res is None:
        res = oracle_port_ms(plain, wrank, TP_WORLD, lanes, args.steps)
        kind = "port"
    value = res["mean_ms"]
    lanes4 = reference_materialize_ms(plain, wrank, TP_WORLD, 4, 3, 1)
    full = reference_load_ms(plain, wrank, TP_WORLD, lanes, 3)
    full4 = reference_load_ms(plain, wrank, TP_WORLD, 4, 3)
    serve = reference_serve_ms(plain, wrank, TP_WORLD, lanes, 2)
    line = {
        "impl": "reference",
        "metric": "graph-set materialization ms (cold start); relocation GB/s vs HBM peak",
        "value": value, "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup if kind == "reference" else 1,
        "ms_per_step": value, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic",
        "config": bench_config(args.workload, plain, wrank),
        "cpu_baseline": {"value": value, "unit": "ms", "cores": lanes, "kind": kind, "cpu_model": cpu_model(),
                         "sample": "reference verify_archive_integrity (single-threaded, pipeline.cpp:411-417) "
                                   "+ PrepareFn over all member graphs on %d prepare lanes (archive written by "
                                   "the reference's own save), %d reps after %d warm-up"
                                   % (lanes, args.steps, args.warmup if kind == "reference" else 1),
                         "integrity_ms": res.get("integrity_best_ms"),
                         "prepare_lanes_4_ms": lanes4["mean_ms"] if lanes4 else None},
        "e2e": {"value": value, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "full_load": {"value": full["mean_ms"] if full else None, "unit": "ms", "prepare_lanes": lanes,
                      "prepare_lanes_4_ms": full4["mean_ms"] if full4 else None,
                      "api": "reference foundry::load (pipeline.cpp:447-557), simulated driver"},
        "serve_replay_all": None if serve is None else {
            "ms": serve["mean_ms"], "us_per_batch": serve["us_per_batch"], "batches": serve["batches"],
            "api": "reference ServingContext::replay of every batch in label order (serve + simulated "
                   "launch, pipeline.cpp:566-569, 876-889)"},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    grank, gworld, local = dist_env()
    if args.impl == "reference":
        run_reference(args, grank, gworld)
        return

    import torch

    import paper_2604_06664_b200 as foundry
    from paper_2604_06664_b200 import capi
    from paper_2604_06664_b200.multirank import RankGroup, distribute_store, tp_rank

    # FOUNDRY_BENCH_SHARED_GPU=1 (testing the N>1 path on a one-GPU box): every
    # rank runs on cuda:0 and the plumbing goes over gloo (NCCL refuses two
    # ranks on one device). The driver's runs never set it.
    shared = os.environ.get("FOUNDRY_BENCH_SHARED_GPU") == "1"
    gpu = 0 if shared else local  # the device this rank drives; `local` still names the node-local rank
    # cold start as the paper measures it (N=1, before this process touches CUDA,
    # so no other context shares the GPU): fresh `foundry load` processes
    cold = cold_process_load(args, gpu) if gworld == 1 and not args.skip_load else {}
    torch.cuda.set_device(gpu)
    group = RankGroup(grank, gworld, local)
    group.init("gloo" if shared else "nccl")
    barrier, reduce_max = group.barrier, group.max

    archive, plain = prepare_archives(args.workload, local, barrier)
    wrank = tp_rank(grank)
    with open(os.path.join(archive, "manifest")) as f:
        manifest = json.load(f)
    base = manifest["allocator"]["base"]
    delta = 0x10000  # exercise K1: the region lands one granule away
    blob = open(os.path.join(archive, "templates.fdt"), "rb").read()
    hdr = capi.store_header(blob)
    alg = capi.algorithmic_bytes(hdr)

    # ---------------- device-resident materialization (value) ----------------
    api = capi.CApi()
    dev = api.device_open(gpu)
    t_fan = time.perf_counter()
    store = distribute_store(group, api, dev, blob, args.fanout)  # the one exchange step
    fanout_ms = (time.perf_counter() - t_fan) * 1e3
    # N > 1: the three SURVEY §8(e) exchange options on the same ranks, each
    # twice after the one above (wall clock from a barrier to the store being
    # resident on this rank, max over ranks)
    fanout_modes = {}
    if gworld > 1:
        for mode in ("ipc", "chain", "host"):
            times = []
            for _ in range(2):
                barrier()
                t_m = time.perf_counter()
                extra = distribute_store(group, api, dev, blob, mode)
                times.append((time.perf_counter() - t_m) * 1e3)
                barrier()  # no rank frees a store a peer may still read
                api.lib.fdy_store_free(extra)
            fanout_modes[mode] = reduce_max(min(times))
    members, _ = api.materialize(dev, store, wrank, TP_WORLD, base + delta)
    flush_w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # each > 126 MB L2
    flush_r = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")

    def flush_l2():
        # a write pass evicts our inputs; a read pass then writes back its
        # dirty lines, so the timed launch starts with a clean, unrelated L2
        flush_w.zero_()
        torch.count_nonzero(flush_r)
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        flush_l2()
        api.materialize(dev, store, wrank, TP_WORLD, base + delta, members)
    sampler = ClockSampler(gpu)
    with sampler:
        barrier()
        torch.cuda.synchronize()
        times = []
        for _ in range(args.steps):
            flush_l2()  # between timed iterations, outside the events
            _, ms = api.materialize(dev, store, wrank, TP_WORLD, base + delta, members)
            times.append(ms)
        torch.cuda.synchronize()
        barrier()
        kernel_ms = statistics.mean(times)
        kernel_ms_max = reduce_max(kernel_ms)
        # the dominant kernel alone (roofline): the same materialization with the
        # relocation grid and the member pass as separate launches, timed apart
        split = []
        for _ in range(args.steps):
            flush_l2()
            split.append(api.materialize_split(dev, store, wrank, TP_WORLD, base + delta, members))
        torch.cuda.synchronize()
        barrier()
        reloc_ms = reduce_max(statistics.mean(r for r, _ in split))
        member_ms = reduce_max(statistics.mean(m for _, m in split))
        # what writing an output of this size alone takes on this GPU (the
        # member pass is write-dominated: 147 MB written, ~17 MB read), same
        # protocol (L2 flushed, CUDA events): a plain st.global.v4 fill of the
        # same arena (fdy_members_write_probe, measurement only); the arena is
        # re-materialized afterwards
        fill_times = []
        for _ in range(args.steps):
            flush_l2()
            fms = ctypes.c_float()
            api.check(api.lib.fdy_members_write_probe(members, ctypes.byref(fms)))
            fill_times.append(fms.value)
        write_ceiling_ms = reduce_max(statistics.mean(fill_times))
        api.materialize(dev, store, wrank, TP_WORLD, base + delta, members)

        # the same on a model-shaped (tier-S) arena of the headline set: 1720-byte
        # GEMM-like argument blocks make the member images ~330 MB (SURVEY §8(d):
        # GB/s is most meaningful on arenas of hundreds of MB)
        ts = None
        if not args.skip_tier_s:
            ts_arch = tier_s_archive(archive) if local == 0 else None
            barrier()
            ts_arch = ts_arch or os.path.join(os.path.dirname(archive), "tier_s")
            ts_blob = open(os.path.join(ts_arch, "templates.fdt"), "rb").read()
            ts_hdr = capi.store_header(ts_blob)
            ts_alg = capi.algorithmic_bytes(ts_hdr)
            ts_store = api.store_upload(dev, ts_blob)
            ts_members, _ = api.materialize(dev, ts_store, wrank, TP_WORLD, base + delta)
            ts_whole, ts_split = [], []
            for _ in range(args.warmup):
                flush_l2()
                api.materialize(dev, ts_store, wrank, TP_WORLD, base + delta, ts_members)
            for _ in range(args.steps):
                flush_l2()
                ts_whole.append(api.materialize(dev, ts_store, wrank, TP_WORLD, base + delta, ts_members)[1])
                flush_l2()
                ts_split.append(api.materialize_split(dev, ts_store, wrank, TP_WORLD, base + delta,
                                                      ts_members)[1])
            torch.cuda.synchronize()
            ts_ms = reduce_max(statistics.mean(ts_whole))
            ts_member_ms = reduce_max(statistics.mean(ts_split))
            api.lib.fdy_members_free(ts_members)
            api.lib.fdy_store_free(ts_store)
            ts = {"workload": args.workload + "~ tier-S (model-shaped argument blocks), rank %d of 8" % wrank,
                  "member_image_bytes": ts_hdr["members_image_bytes"], "store_bytes": len(ts_blob),
                  "ms": ts_ms, "member_pass_ms": ts_member_ms,
                  "member_pass_algorithmic_bytes": ts_alg["member_pass"],
                  "member_pass_gbps": ts_alg["member_pass"] / (ts_member_ms * 1e-3) / 1e9,
                  "whole_launch_gbps": ts_alg["total"] / (ts_ms * 1e-3) / 1e9}

        # ------- end to end through the C-ABI: archive files -> host result -------
        # fdy_prepare_archive = read every file, DMA to HBM, GPU CRC of every
        # file vs the manifest, fused kernel over every member, copy all member
        # images back to (pinned) host memory.
        lanes = max(1, (os.cpu_count() or 4) // gworld)  # the host cores are shared by the ranks
        host_out = api.host_alloc(dev, hdr["members_image_bytes"])
        for _ in range(2):  # warm-up: page cache + pinned staging pool
            api.prepare_archive(dev, archive, wrank, TP_WORLD, base + delta, lanes, host_out,
                                hdr["members_image_bytes"])
        e2e_times, e2e_parts = [], []
        for _ in range(args.e2e_steps):
            barrier()
            t0 = time.perf_counter()
            parts = api.prepare_archive(dev, archive, wrank, TP_WORLD, base + delta, lanes, host_out,
                                        hdr["members_image_bytes"])
            e2e_times.append((time.perf_counter() - t0) * 1e3)
            e2e_parts.append(parts)
        e2e_ms = reduce_max(statistics.mean(e2e_times))
        # the same call on the archive as the reference writes it (no
        # templates.fdt): graphs.bin goes to HBM and the GPU packer
        # (kernels/pack.cu) builds the template store before the kernel runs
        for _ in range(2):
            api.prepare_archive(dev, plain, wrank, TP_WORLD, base + delta, lanes, host_out,
                                hdr["members_image_bytes"])
        plain_times, plain_parts = [], []
        for _ in range(args.e2e_steps):
            barrier()
            t0 = time.perf_counter()
            parts = api.prepare_archive(dev, plain, wrank, TP_WORLD, base + delta, lanes, host_out,
                                        hdr["members_image_bytes"])
            plain_times.append((time.perf_counter() - t0) * 1e3)
            plain_parts.append(parts)
        e2e_plain_ms = reduce_max(statistics.mean(plain_times))
        api.lib.fdy_host_free(host_out)

        # ------- LOAD to every graph servable through the Python API -------
        servable = {}
        if not args.skip_load:
            servable["share_execs"] = full_load_stats(foundry, archive, wrank, lanes, args.load_steps, barrier,
                                                      reduce_max, share_execs=True)
            servable["per_template"] = full_load_stats(foundry, archive, wrank, lanes, args.load_steps, barrier,
                                                       reduce_max)
            # the archive as the reference writes it: the store is packed on the GPU at LOAD
            servable["reference_written"] = full_load_stats(foundry, plain, wrank, lanes, args.load_steps,
                                                            barrier, reduce_max, share_execs=True)
        # serve sweeps (reference ServingSet::serve, templater.cpp:177-188): apply every
        # batch's parameters in label order; then serve + replay every batch, the
        # reference's `bench --mode load` loop (pipeline.cpp:876-889)
        serve_ms = {}
        if not args.skip_load:
            for mode in ("per_template", "shared_execs", "device_updates"):
                h = foundry.load(archive, rank=wrank, world=TP_WORLD, prepare_lanes=lanes,
                                 share_execs=mode == "shared_execs", device_updates=mode == "device_updates")
                bs = h.batches()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                touched = sum(h.serve(b) for b in bs)
                torch.cuda.synchronize()  # device_updates queues its serve kernels: count them
                ms = (time.perf_counter() - t0) * 1e3
                t0 = time.perf_counter()
                for b in bs:
                    h.replay(b)  # serve + launch + device-side trace verification
                replay_ms = (time.perf_counter() - t0) * 1e3
                serve_ms[mode] = {"ms": ms, "us_per_serve": ms * 1e3 / len(bs), "batches": len(bs),
                                  "nodes_touched": touched, "serve_replay_all_ms": replay_ms,
                                  "replay_verified": True}
                h.close()
    clocks = sampler.summary()

    api.lib.fdy_members_free(members)
    api.lib.fdy_store_free(store)
    api.lib.fdy_device_close(dev)

    if grank != 0:
        group.close()
        return

    peak, peak_src = hbm_peak()
    achieved = alg["member_pass"] / (member_ms * 1e-3) / 1e9  # the dominant kernel
    launch_gbps = alg["total"] / (kernel_ms_max * 1e-3) / 1e9     # the whole materialization
    prof = os.path.join(ROOT, "profiles", "materialize_ncu_summary.json")
    traffic = None
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    ep = {k: statistics.mean(p[k] for p in e2e_parts) for k in e2e_parts[0]}

    # ---------------- CPU baseline: the reference itself, rank 0, N=1 ----------------
    cpu = None
    refarch = reference_archive(args.workload) or plain
    if not args.no_cpu_baseline and gworld == 1:
        refm = reference_materialize_ms(refarch, wrank, TP_WORLD, lanes, 5)
        if refm is not None:
            refm4 = reference_materialize_ms(refarch, wrank, TP_WORLD, 4, 3)
            refl = reference_load_ms(refarch, wrank, TP_WORLD, lanes, 3)
            refl4 = reference_load_ms(refarch, wrank, TP_WORLD, 4, 3)
            refs = reference_serve_ms(refarch, wrank, TP_WORLD, lanes, 2)
            cpu = {"value": refm["mean_ms"], "unit": "ms", "cores": lanes, "kind": "reference",
                   "cpu_model": cpu_model(),
                   "sample": "reference verify_archive_integrity + PrepareFn over all 512 members "
                             "(rank 0 of 8, %d prepare lanes; archive written by the reference's save), "
                             "5 reps after 1 warm-up" % lanes,
                   "reference_integrity_ms": refm["integrity_best_ms"],
                   "reference_prepare_lanes_4_ms": refm4["mean_ms"] if refm4 else None,
                   "reference_full_load_ms": refl["mean_ms"] if refl else None,
                   "reference_full_load_lanes_4_ms": refl4["mean_ms"] if refl4 else None,
                   "reference_serve_replay_all_ms": refs["mean_ms"] if refs else None}
        else:
            port = oracle_port_ms(plain, wrank, TP_WORLD, lanes, 3)
            cpu = {"value": port["mean_ms"], "unit": "ms", "cores": lanes, "kind": "port",
                   "sample": "oracle/foundry_oracle.c materialization of every member, 3 reps"}

    graphs = hdr["n_members"]
    line = {
        "metric": "graph-set materialization ms (cold start); relocation GB/s vs HBM peak",
        "value": kernel_ms_max,
        "unit": "ms",
        "n_gpus": gworld,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": kernel_ms_max,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic",
        "config": bench_config(args.workload, archive, wrank),
        "store": {"store_bytes": len(blob), "member_image_bytes": hdr["members_image_bytes"],
                  "relocation_delta": delta, "nodes": hdr["total_nodes"], "templates": hdr["n_groups"]},
        "graphs_per_s": gworld * graphs / (kernel_ms_max * 1e-3),
        "nodes_per_s": gworld * hdr["total_nodes"] / (kernel_ms_max * 1e-3),
        "relocation_gbps": launch_gbps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     # what the DRAM counters of the ncu capture (profiles/) say the same
                     # launch moved, over the same event time: below `frac` when part of
                     # the output is still dirty in the 126 MB L2 when the kernel ends
                     "frac_dram": (traffic / (member_ms * 1e-3) / 1e9 / peak) if traffic else None,
                     # a plain fill of the member-image size on the same GPU, same
                     # protocol: the write-only floor of a launch this size
                     "write_ceiling": {"ms": write_ceiling_ms, "bytes": hdr["members_image_bytes"],
                                       "gbps": hdr["members_image_bytes"] / (write_ceiling_ms * 1e-3) / 1e9,
                                       "member_pass_over_write_floor": member_ms / write_ceiling_ms},
                     "algorithmic_bytes": alg["member_pass"],
                     "kernel": "fdy_materialize_kernel (member pass: K2 diff + K1 relocated lanes + "
                               "K3 rank patch), CUDA events around it alone, L2 flushed",
                     "kernel_ms": member_ms,
                     "relocation_prepass": {"kernel": "fdy_relocate_templates_kernel (3.4 MB of "
                                                      "templates, once per launch)", "ms": reloc_ms},
                     "whole_launch": {"ms": kernel_ms_max, "algorithmic_bytes": alg["total"],
                                      "achieved": launch_gbps, "frac": launch_gbps / peak,
                                      "note": "both grids under programmatic dependent launch = value"}},
        "e2e": {"value": e2e_ms, "unit": "ms",
                "h2d_bytes_per_step": int(ep["h2d_bytes"]),
                "d2h_bytes_per_step": int(ep["d2h_bytes"]),
                "steps": args.e2e_steps,
                "api": "C-ABI fdy_prepare_archive (include/foundry_b200.h): archive files -> GPU "
                       "integrity + fused materialization -> all member images in host memory",
                # (the store's CRC blocks run interleaved with its DMA pieces on a side
                # stream: no separate kernel time, see profiles/ for the launch list)
                "breakdown": {k: v for k, v in ep.items() if k.endswith("_ms") and k != "crc_kernel_ms"}},
        "e2e_plain": {"value": e2e_plain_ms, "unit": "ms",
                      "min": min(plain_times), "max": max(plain_times),
                      "h2d_bytes_per_step": int(statistics.mean(p["h2d_bytes"] for p in plain_parts)),
                      "d2h_bytes_per_step": int(statistics.mean(p["d2h_bytes"] for p in plain_parts)),
                      "steps": args.e2e_steps,
                      "api": "C-ABI fdy_prepare_archive on the archive as the reference writes it (no "
                             "templates.fdt): graphs.bin DMAed to HBM, the GPU packer (kernels/pack.cu: "
                             "record walk, validation, kernel-key table, images, ballot/scan diff "
                             "compaction) builds the template store, then the same fused materialization",
                      "breakdown": {k: statistics.mean(p[k] for p in plain_parts) for k in plain_parts[0]
                                    if k.endswith("_ms") and k != "crc_kernel_ms"}},
        "e2e_servable": None if not servable else dict(
            servable["share_execs"],
            api="paper_2604_06664_b200.load(archive, rank, world, share_execs=True): files -> every "
                "template instantiated (one exec per graph shape), every function of every template "
                "loaded, every member's parameters resident in HBM",
            reference_full_load_ms=(cpu or {}).get("reference_full_load_ms"),
            per_template=servable["per_template"],
            reference_written_archive=dict(servable["reference_written"],
                                           note="same LOAD (share_execs) of the archive the reference's "
                                                "save writes (no templates.fdt): graphs.bin to HBM and the "
                                                "GPU packer first (breakdown pack_ms)"),
            floor="driver-serialized: ~11-15 us per function load (9028 functions in 96 libraries) and "
                  "~35 ms per cuGraphInstantiate of a 1036-node template (~50 us per concurrent branch "
                  "node); profiles/round2_driver_floor.md"),
        "tier_s": None if ts is None else dict(ts, member_pass_frac=ts["member_pass_gbps"] / peak,
                                               whole_launch_frac=ts["whole_launch_gbps"] / peak),
        "serve_sweep": serve_ms or None,
        "cold_process_load": None if not cold else {
            "unit": "ms", "per_template": cold.get("per_template"), "share_execs": cold.get("share_execs"),
            "cuda_init_only": cold.get("cuda_init"), "process_exit": cold.get("process_exit"),
            "device_open_ms": cold.get("device_open_ms"), "load_after_device_open_ms": cold.get("load_ms"),
            "what": "wall clock of `foundry load --archive <headline> --rank r --world 8` in a fresh "
                    "process from exec to its 'ready' line: CUDA context creation + LOAD to every "
                    "template servable (the paper's cold start); cuda_init_only = a fresh process "
                    "that only opens the device (CUDA context creation, until exit); process_exit = "
                    "exec to exit, teardown included; median/min/max of 5 interleaved rounds. The "
                    "reference arm's simulated LOAD creates no CUDA context"},
        "cpu_baseline": cpu,
        "clocks": clocks,
        # per timed step: the gate kernel that holds the stream while the launches are
        # submitted (its hold ends before the start event), the relocation grid, the member grid
        "gpu_launches": args.steps * (3 if delta else 2),
        "fanout": {"mode": args.fanout if gworld > 1 else "none", "ms": fanout_ms,
                   "modes_ms": fanout_modes or None,
                   "store_bytes": len(blob)},
    }
    print(json.dumps(line), flush=True)
    group.close()


if __name__ == "__main__":
    main()
