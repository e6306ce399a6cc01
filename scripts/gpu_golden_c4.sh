#!/bin/bash
# C4 (n=2^32 DNA) golden checksums from the unmodified reference (baseline/_ref)
# on the GPU box's host (needs ~100 GB RAM), then the GPU parity suites.
set -x
nproc; free -g | head -2
( python tests/golden/make_golden_large.py --out=gpurun_out/golden_c4.json C4 ) > gpurun_out/golden_c4.log 2>&1
echo "golden rc=$?"
tail -5 gpurun_out/golden_c4.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
