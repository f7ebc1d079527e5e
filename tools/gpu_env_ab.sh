# A/B of environment-variable hooks on the headline: usage gpu_env_ab.sh "VAR=val" "VAR=val" ...
cfg=${CFG:-rm29_L4_M20}
for i in 1 2; do
for e in "$@"; do
  env $e timeout 300 python bench.py --no-cpu --config $cfg > gpurun_out/env.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/env.log').read().strip().splitlines()[-1]);print(sys.argv[1],round(d['value']),round(d['decode_only']['value']))" "$e"
done; done
