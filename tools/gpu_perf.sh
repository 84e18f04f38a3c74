#!/bin/bash
# Timing only (no parity suite): per-order 2D step times + the parity file for the kernel.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/prof_step.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
for m in 2 3 4 5 6 7 8; do timeout 120 python tools/prof_step.py --m $m --n 1024 --steps 4 >> gpurun_out/prof_step.txt 2>&1; done
for m in 3 4 5 8; do timeout 120 python tools/prof_step.py --scheme cons --m $m --n 2048 --steps 4 --walls >> gpurun_out/prof_step.txt 2>&1; done
