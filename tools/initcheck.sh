#!/bin/bash
# compute-sanitizer initcheck (reads of uninitialized device memory) over the
# kernels that run without VMM reservations: fused materialize, GPU CRC,
# fdy_prepare_archive on both archive layouts (staging + GPU packer), the GPU
# packer alone, the chain fan-out (tools/_sanitize_case.py --no-load).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
D=$(mktemp -d)
python tools/_sanitize_case.py --prepare $D
timeout 1200 $S --tool initcheck --print-limit 1000000 --error-exitcode 9 "$(command -v python)" tools/_sanitize_case.py --no-load $D > gpurun_out/san_initcheck.txt 2>&1; echo "initcheck rc=$?"
python tools/_initcheck_summary.py gpurun_out/san_initcheck.txt > gpurun_out/san_initcheck_summary.txt; rm -f gpurun_out/san_initcheck.txt; cat gpurun_out/san_initcheck_summary.txt

