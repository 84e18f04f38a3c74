#!/bin/bash
# One iteration: GPU parity tests, per-order timing, then an ncu capture of one launch.
#   tools/gpu_iter.sh <tag> <prof_step.py args for ncu...>
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=$1; shift
bash tools/gpu_quick.sh
grep -q "pytest rc=0" gpurun_out/pytest_gpu.log && bash tools/gpu_ncu.sh $tag "$@"
