# A/B of library variants (tools/ablate.py), 3 alternating rounds; extra args after --
#   bash tools/gpu_ab.sh [--c4] -- libsbattn.so libsbattn_x.so ...
set -x
mkdir -p gpurun_out
opts=""
while [ "$1" != "--" ] && [ -n "$1" ]; do opts="$opts $1"; shift; done
shift
for i in 1 2 3; do
  for v in "$@"; do timeout 120 python tools/ablate.py paper_2410_17980_b200/$v $opts; done
done > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log | grep fwd
