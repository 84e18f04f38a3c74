#!/bin/bash
# ncu --set full capture of one cell-map launch:  tools/gpu_ncu.sh <tag> <prof_step.py args...>
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=$1; shift
timeout 300 python tools/prof_step.py "$@" --steps 3 > gpurun_out/plain_$tag.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cellmap -s 1 -c 1 -o gpurun_out/prof_$tag \
  python tools/prof_step.py "$@" --steps 3 > gpurun_out/ncu_$tag.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$tag.log
