# A/B: lock-step barrier options of the throughput kernel (headline), decode-only and step rate
for i in 1 2; do
for opt in "" "--lockstep 8" "--lockstep 4" "--no-lockstep"; do
  timeout 300 python bench.py --no-cpu $opt > gpurun_out/ls.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/ls.log').read().strip().splitlines()[-1]);print(sys.argv[1] or 'cta',round(d['value']),round(d['decode_only']['value']))" "$opt"
done; done
