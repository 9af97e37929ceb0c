# Round-end evidence run (one gpurun call): bench line, launch list, ncu captures.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc $?"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --cfg5-events 2000 --cfg3-events 512 > gpurun_out/plain_bench_small.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --cfg5-events 2000 --cfg3-events 512 > gpurun_out/ncu_bench.log 2>&1; echo "ncu bench rc $?"
python tools/prof_kernels.py events > gpurun_out/plain_ev.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:damf_ppr_kernel -s 20 -c 1 -o gpurun_out/pprk_final python tools/prof_kernels.py events > gpurun_out/ncu_pprk.log 2>&1; echo "ncu pprk rc $?"
