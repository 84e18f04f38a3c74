#!/bin/bash
# Race / bounds stress (tools/race_stress.py): the product build once, the
# HW_CM_DEBUG build (slot poisoning, random delays, bounds traps) three times,
# all bitwise compared; then the parity suites under the debug build.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
out=gpurun_out/race_stress.txt
: > $out
timeout 600 python tools/race_stress.py --out /tmp/rs_default.npz >> $out 2>&1; echo "default rc=$?" >> $out
for i in 1 2 3; do
  HERMB200_LIB=build_var/debug/libhermb200.so timeout 900 python tools/race_stress.py --out /tmp/rs_debug$i.npz >> $out 2>&1
  echo "debug run $i rc=$?" >> $out
done
python tools/race_stress.py --compare /tmp/rs_default.npz /tmp/rs_debug1.npz /tmp/rs_debug2.npz /tmp/rs_debug3.npz >> $out 2>&1
echo "compare rc=$?" >> $out
HERMB200_LIB=build_var/debug/libhermb200.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_interior.py \
  tests/test_c3.py tests/test_gpu_slab.py tests/test_energy_cons2d.py -m gpu -q >> $out 2>&1
echo "debug-build parity rc=$?" >> $out
