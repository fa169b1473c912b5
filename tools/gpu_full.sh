# full round measurement: parity tests, smoke, bench (contract line), C3 skip report, C4 varlen,
# ncu, C2 strong scaling, C5 training step
set -x
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 600 python tests/reports/c3_skip_report.py --out gpurun_out/c3_skip.json > gpurun_out/skip.log 2>&1
for n in 2 4 8; do timeout 200 python tools/varlen_bench.py --simulate-ranks $n; done > gpurun_out/c4.log 2>&1
bash tools/gpu_ncu.sh
timeout 300 python tools/strong_scaling.py > gpurun_out/c2_strong.log 2>&1
timeout 400 python tools/c5_train_step.py > gpurun_out/c5.log 2>&1
for f in bench bench_ref skip smoke pytest_gpu c2_strong c5; do tail -n 2 gpurun_out/$f.log; done
