cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./tools/dmma_sweep > gpurun_out/dmma_sweep.jsonl 2>&1
for m in 4 6 8; do python tools/prof_step.py --m $m --n 1024 --steps 4 >> gpurun_out/prof_step.txt 2>&1; done
python tools/prof_step.py --m 4 --n 1024 --steps 3 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:cellmap -s 1 -c 1 -o gpurun_out/prof_m4 python tools/prof_step.py --m 4 --n 1024 --steps 3 > gpurun_out/ncu.log 2>&1
