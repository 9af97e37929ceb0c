set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; echo "bench rc $?"
python tools/prof_mat.py 256 > gpurun_out/plain256.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:materialize_bf16 -s 1 -c 1 -o gpurun_out/mat256b python tools/prof_mat.py 256 > gpurun_out/ncu256b.log 2>&1; echo "ncu256 rc $?"
python tools/prof_mat.py 128 > gpurun_out/plain128.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:materialize_tc128 -s 1 -c 1 -o gpurun_out/mat128b python tools/prof_mat.py 128 > gpurun_out/ncu128b.log 2>&1; echo "ncu128 rc $?"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --cfg5-events 2000 --cfg3-events 512 > gpurun_out/plain_bench_small.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --cfg5-events 2000 --cfg3-events 512 > gpurun_out/ncu_bench.log 2>&1; echo "ncu bench rc $?"
