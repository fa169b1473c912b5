# ncu full capture of the three sb_ kernels (one launch each) + launch list
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sb_ -s 3 -c 3 -o gpurun_out/full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-sdpa > gpurun_out/ncu_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sb_ -c 15 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-sdpa > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/ncu_full.log
