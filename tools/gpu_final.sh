# round-2 final measurement: parity tests, smoke, sanitizers, bench (contract line +
# reference arm), C3 skip report, C4 varlen (+ simulated ranks), ncu (C2 and C4),
# C2 strong scaling, C5 training step
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rA --durations=10 2>&1 | tail -150 > gpurun_out/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for t in memcheck racecheck synccheck; do for m in "" --many; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_case.py $m > gpurun_out/san_${t}$m.log 2>&1
  echo "$t $m: $(tail -1 gpurun_out/san_${t}$m.log)" >> gpurun_out/sanitizer.txt
done; done
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 900 python tests/reports/c3_skip_report.py --check-heads 1 --out gpurun_out/c3_skip.json > gpurun_out/skip.log 2>&1
for n in 1 2 4 8; do timeout 300 python tools/varlen_bench.py --simulate-ranks $n; done > gpurun_out/c4.log 2>&1
bash tools/gpu_ncu.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sb_ -s 3 -c 3 -o gpurun_out/c4_full -f python tools/ablate.py paper_2410_17980_b200/libsbattn.so --c4 > gpurun_out/ncu_c4.log 2>&1
timeout 600 python tools/strong_scaling.py > gpurun_out/c2_strong.log 2>&1
timeout 600 python tools/c5_train_step.py > gpurun_out/c5.log 2>&1
for f in bench bench_ref skip smoke c2_strong c5 c4; do echo "== $f"; tail -n 3 gpurun_out/$f.log | cut -c1-600; done
cat gpurun_out/sanitizer.txt
grep -E "passed|failed" gpurun_out/pytest_gpu.log
