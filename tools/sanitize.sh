#!/bin/bash
# compute-sanitizer over the kernels on small archives: memcheck on the whole
# LOAD + replay + serve path (smoke), racecheck / synccheck on the fused
# materialize kernel and the CRC kernels (C-ABI, tools/_sanitize_case.py).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
D=$(mktemp -d)
python tools/_sanitize_case.py --prepare $D   # archives written outside the sanitizer
$S --tool memcheck --leak-check no --error-exitcode 9 python tools/_sanitize_case.py $D > gpurun_out/san_memcheck.txt 2>&1; echo "memcheck rc=$?"
$S --tool racecheck --error-exitcode 9 python tools/_sanitize_case.py $D > gpurun_out/san_racecheck.txt 2>&1; echo "racecheck rc=$?"
$S --tool synccheck --error-exitcode 9 python tools/_sanitize_case.py $D > gpurun_out/san_synccheck.txt 2>&1; echo "synccheck rc=$?"
# (initcheck: the sanitizer itself segfaults on this process — VMM reservations — so it is not run)
for f in gpurun_out/san_*.txt; do echo "== $f"; tail -2 "$f"; done
