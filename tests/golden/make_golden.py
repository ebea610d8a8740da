"""Regenerates tests/golden/golden.json from the compiled reference.

Run in the container that has /root/reference (after `make -C oracle ref`):

    python tests/golden/make_golden.py

Every value comes from the UNMODIFIED reference (oracle/_ref/ref_tool):
  * file digests of reference-written archives (`save`),
  * CRC-64 of the SAVE-time traces,
  * per-member CRC-64 of the reference PrepareFn output (`prepare`:
    parse_graph_at + apply_rank_patches) for several (rank, world),
  * for relocation (no reference function): the CRC of the reference replay
    traces of oracle-relocated members at the shifted base (`replay`), i.e.
    the reference simulated driver's verdict on the relocated graphs.
The fixtures let the oracle and the product be pinned without the reference.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import fndg  # noqa: E402
from oracle_lib import Oracle  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
SPECS = {
    "micro": "micro",
    "moe-small": "seed = 13\nbatch_max = 12\nlayers = 12\nkernels_per_layer = 8\nthresholds = 5,9\n"
                 "hidden_offset_density = 0.5\ncomm = spmd\ncollectives_per_layer = 2\n"
                 "kv_cache_bytes = 16777216\nweights_bytes_per_layer = 262144\nio_bytes = 65536\n"
                 "scratch_bytes_per_batch = 8192\n",
    "llama3-8b": os.path.join(ROOT, "paper_2604_06664_b200", "workloads", "llama3-8b.spec"),
}
CASES = [(0, 1, 0), (1, 2, 0), (3, 4, 0), (0, 1, 0x10000), (2, 4, 0x10000000000)]


def main() -> None:
    oracle = Oracle(os.path.join(ROOT, "oracle", "_build", "liboracle.so"))
    out = {"crc64_check": {"123456789": "%016x" % oracle.crc64(b"123456789")}, "archives": {}}
    with tempfile.TemporaryDirectory() as tmp:
        for name, spec in SPECS.items():
            spec_file = spec
            if "\n" in spec:
                spec_file = os.path.join(tmp, name + ".spec")
                open(spec_file, "w").write(spec)
            arch = os.path.join(tmp, name)
            traces = os.path.join(tmp, name + ".traces")
            subprocess.run([REF, "save", spec_file, arch, traces], check=True, capture_output=True)
            m = json.load(open(os.path.join(arch, "manifest")))
            entry = {
                "spec": open(spec_file).read() if os.path.exists(spec_file) else spec,
                "files": {k: "%016x" % v for k, v in m["files"].items()},
                "manifest_crc": "%016x" % oracle.crc64(open(os.path.join(arch, "manifest"), "rb").read()),
                "save_traces_crc": "%016x" % oracle.crc64(open(traces, "rb").read()),
                "cases": [],
            }
            for rank, world, delta in CASES:
                case = {"rank": rank, "world": world, "delta": delta}
                if delta == 0:
                    prep = os.path.join(tmp, "prep.fndg")
                    subprocess.run([REF, "prepare", arch, str(rank), str(world), prep], check=True)
                    data = open(prep, "rb").read()
                    case["source"] = "reference prepare"
                else:
                    data, nreloc = oracle.materialize_archive(arch, rank, world, delta)
                    prep = os.path.join(tmp, "reloc.fndg")
                    open(prep, "wb").write(data)
                    rt = os.path.join(tmp, "reloc.traces")
                    subprocess.run([REF, "replay", arch, prep, "%x" % delta, rt], check=True)
                    case["source"] = "oracle relocation, accepted by reference replay"
                    case["reference_replay_traces_crc"] = "%016x" % oracle.crc64(open(rt, "rb").read())
                    case["relocated_slots"] = nreloc
                case["container_crc"] = "%016x" % oracle.crc64(data)
                case["records"] = {str(lab): "%016x" % oracle.crc64(rec)
                                   for lab, rec in fndg.records(data).items()}
                entry["cases"].append(case)
            out["archives"][name] = entry
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
