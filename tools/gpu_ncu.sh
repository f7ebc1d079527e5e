# one ncu --set full capture of the headline decode kernel (source-level)
cfg=${1:-rm29_L4_M20}
tag=${2:-dk2}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel2 -s 2 -c 1 -o gpurun_out/$tag python bench.py --steps 1 --warmup 1 --no-cpu --config $cfg > gpurun_out/ncu_$tag.log 2>&1; echo ncu exit $?
