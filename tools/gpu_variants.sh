# decode-only bench of the working library and each tools/_ab/librmfht_<v>.so variant
cfg=${CFG:-rm29_L4_M20}
for v in base "$@"; do
  for i in 1 2; do
    if [ "$v" = base ]; then lib=$PWD/paper_2108_12550_b200/librmfht.so; else lib=$PWD/tools/_ab/librmfht_$v.so; fi
    RMFHT_LIB_OVERRIDE=$lib timeout 300 python bench.py --no-cpu --config $cfg > gpurun_out/var_$v.log 2>&1
    python -c "import json,sys;d=json.loads(open('gpurun_out/var_$v.log').read().strip().splitlines()[-1]);print('$v',d['value'],d['decode_only']['value'])" || tail -3 gpurun_out/var_$v.log
  done
done
