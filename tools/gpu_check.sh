set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest exit $?
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo bench exit $?
tail -1 gpurun_out/bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel2 -s 2 -c 1 -o gpurun_out/dk2 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu.log 2>&1; echo ncu exit $?
