# round 2 probe: MUFU single-warp rate ubench; C4 (d=64) per-phase times + ncu of the d=64 kernels
set -x
mkdir -p gpurun_out
./tools/ubench/ub_mufu > gpurun_out/ub_mufu.txt 2>&1
timeout 300 python tools/varlen_bench.py --steps 10 > gpurun_out/c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sb_ -s 3 -c 3 -o gpurun_out/c4_full -f python tools/varlen_bench.py --steps 1 --warmup 1 > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/ncu_c4.log
cat gpurun_out/ub_mufu.txt
tail -5 gpurun_out/c4.log
