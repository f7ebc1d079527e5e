# every BASELINE config: bench line with the start-of-session library and the working one (decode-only A/B)
for cfg in rm29_L4_M20 rm27_L2_M4 rm37_L8_M32 rm29_L1_M512 rm25_fhtfsc rm29_autssc_P512; do
  RMFHT_LIB_OVERRIDE=$PWD/tools/_ab/librmfht_base.so timeout 300 python bench.py --no-cpu --config $cfg > gpurun_out/old_$cfg.json 2>gpurun_out/old_$cfg.err
  timeout 300 python bench.py --no-cpu --config $cfg > gpurun_out/new_$cfg.json 2>gpurun_out/new_$cfg.err
  python - "$cfg" <<'PY'
import json,sys
c=sys.argv[1]
def g(f):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); return d['value'], d['decode_only']['value'], d['roofline']['frac']
    except Exception as e: return str(e)
print(c, 'old', g(f'gpurun_out/old_{c}.json'), 'new', g(f'gpurun_out/new_{c}.json'))
PY
done
