# round profile: launch list of the headline bench + one ncu --set full capture of the decode kernel
tag=${1:-r1_v18}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/${tag}_launch_run.log 2>&1; echo launches exit $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel2 -s 2 -c 1 -o gpurun_out/${tag}_dk2 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/${tag}_ncu.log 2>&1; echo ncu exit $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sample_kernel -s 1 -c 1 -o gpurun_out/${tag}_sample python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/${tag}_ncu_s.log 2>&1; echo ncu2 exit $?
