# round measurement: GPU tests, smoke, every config's bench line, the reference arm
tag=${1:-r1_v18}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo pytest exit $?
timeout 300 python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.log 2>&1; echo smoke exit $?
for cfg in rm29_L4_M20 rm27_L2_M4 rm37_L8_M32 rm29_L1_M512 rm25_fhtfsc rm29_autssc_P512; do
  timeout 600 python bench.py --config $cfg > gpurun_out/${tag}_bench_$cfg.json 2> gpurun_out/${tag}_bench_$cfg.err; echo $cfg exit $?
done
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_reference_arm.json 2> gpurun_out/${tag}_bench_reference_arm.err; echo ref exit $?
