# A/B: run GPU tests on the working library, then bench base vs new (headline)
cfg=${1:-rm29_L4_M20}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest exit $?; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do
RMFHT_LIB_OVERRIDE=$PWD/tools/_ab/librmfht_base.so timeout 300 python bench.py --no-cpu --config $cfg > gpurun_out/bench_base.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_base.log').read().strip().splitlines()[-1]);print('base',d['value'],d['decode_only']['value'])"
timeout 300 python bench.py --no-cpu --config $cfg > gpurun_out/bench_new.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_new.log').read().strip().splitlines()[-1]);print('new ',d['value'],d['decode_only']['value'])"
done
