#!/bin/bash
# GPU parity tests + per-order timing of the 2D steps.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/prof_step.txt
for m in 2 3 4 5 6 7 8; do timeout 120 python tools/prof_step.py --m $m --n 1024 --steps 4 >> gpurun_out/prof_step.txt 2>&1; done
for m in 4 5 8; do timeout 120 python tools/prof_step.py --scheme cons --m $m --n 2048 --steps 4 --walls >> gpurun_out/prof_step.txt 2>&1; done
