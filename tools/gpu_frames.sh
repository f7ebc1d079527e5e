# decode-only and step rate of the headline at several batch sizes (tail of the lock-step rounds)
for i in 1 2; do
for fr in 16384 15984 32768 31968; do
  timeout 300 python bench.py --no-cpu --frames $fr > gpurun_out/fr.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/fr.log').read().strip().splitlines()[-1]);print($fr,round(d['value']),round(d['decode_only']['value']),round(d['e2e']['value']))" || tail -3 gpurun_out/fr.log
done; done
