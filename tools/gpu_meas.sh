# measurements for DESIGN/profiles: bench (ours + reference arm), C3 report, C4 (+ simulated
# ranks), C2 strong scaling, torchrun 2-rank bench plumbing check (gloo on one GPU)
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 900 python tests/reports/c3_skip_report.py --check-heads 1 --out gpurun_out/c3_skip.json > gpurun_out/skip.log 2>&1
for n in 2 4 8; do timeout 300 python tools/varlen_bench.py --simulate-ranks $n; done > gpurun_out/c4.log 2>&1
timeout 600 python tools/strong_scaling.py > gpurun_out/c2_strong.log 2>&1
SB_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-sdpa > gpurun_out/bench_2.log 2>&1
tail -n 2 gpurun_out/bench_2.log | cut -c1-300
