# round-2 measurement on one B200 (gpurun): GPU tests, smoke, every config's
# bench line, the reference arm, per-config launch lists and one ncu --set full
# capture of each config's dominant kernel.  usage: tools/gpu_round2.sh TAG [quick]
tag=${1:-r2_v1}
o=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $o/${tag}_pytest_gpu.log 2>&1; echo pytest $?
timeout 300 python __graft_entry__.py smoke > $o/${tag}_smoke.log 2>&1; echo smoke $?
for cfg in rm29_L4_M20 rm27_L2_M4 rm37_L8_M32 rm29_L1_M512 rm25_fhtfsc rm29_autssc_P512; do
  timeout 600 python bench.py --config $cfg > $o/${tag}_bench_$cfg.json 2> $o/${tag}_bench_$cfg.err; echo bench $cfg $?
done
timeout 600 python bench.py --impl reference > $o/${tag}_bench_reference_arm.json 2> $o/${tag}_bench_reference_arm.err; echo ref $?
[ "$2" = quick ] && exit 0
for cfg in rm29_L4_M20 rm27_L2_M4 rm37_L8_M32 rm29_L1_M512 rm25_fhtfsc rm29_autssc_P512; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv \
    --log-file $o/${tag}_launches_$cfg.csv python bench.py --steps 1 --warmup 3 --no-cpu --config $cfg > /dev/null 2>&1; echo launches $cfg $?
done
cap() {  # config kernel-regex frames
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o $o/${tag}_ncu_$1 \
    python bench.py --steps 1 --warmup 3 --no-cpu --config $1 --frames $3 > $o/${tag}_ncu_$1.log 2>&1; echo ncu $1 $?
}
cap rm29_L4_M20 decode_kernel2 16384
cap rm27_L2_M4 pair_kernel 65536
cap rm37_L8_M32 decode_kernel2 8192
cap rm29_L1_M512 grp_kernel 1024
cap rm25_fhtfsc lane_kernel 1048576
cap rm29_autssc_P512 aut_ssc 1024
