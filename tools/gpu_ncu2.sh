#!/bin/bash
# ncu captures of the m=4 and m=8 dissipative kernels (one launch each).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
bash tools/gpu_ncu.sh $1_m4 --m 4 --n 1024
bash tools/gpu_ncu.sh $1_m8 --m 8 --n 1024
