# A/B of library variants on the C2 kernels (tools/ablate.py), 3 alternating rounds
set -x
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in "$@"; do timeout 120 python tools/ablate.py paper_2410_17980_b200/$v; done
done > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log | grep fwd
