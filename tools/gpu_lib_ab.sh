# A/B of library variants built by tools/build_variant.py: usage gpu_lib_ab.sh NAME NAME ... ("cur" = the working library)
cfg=${CFG:-rm29_L4_M20}
for i in 1 2; do
for n in "$@"; do
  if [ "$n" = cur ]; then unset RMFHT_LIB_OVERRIDE; else export RMFHT_LIB_OVERRIDE=$PWD/tools/_ab/librmfht_$n.so; fi
  timeout 300 python bench.py --no-cpu --config $cfg > gpurun_out/lib.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/lib.log').read().strip().splitlines()[-1]);print(sys.argv[1],round(d['value']),round(d['decode_only']['value']),d.get('fer_check', d['config'].get('fer_check')))" "$n"
done; done
