# Round-2 evidence run (one gpurun call): tests, bench line, launch lists, ncu captures.
# Outputs under gpurun_out/ (copied into profiles/ by hand after reading them).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc $?"
timeout 1200 python bench.py > gpurun_out/r2_bench_line.json 2> gpurun_out/r2_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err; echo "ref rc $?"
# launch list of the bench's own kernels (headline leg only)
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-sub > gpurun_out/r2_plain_bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'damf|materialize|fold_rows|ppr_|tsvd|gram|spmm' --csv --log-file gpurun_out/r2_bench_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-sub > gpurun_out/r2_ncu_bench.log 2>&1; echo "ncu bench rc $?"
# event kernel at the cfg-5-like steady state
python tools/prof_r2.py cfg5ev > gpurun_out/r2_plain_cfg5ev.log 2>&1
SK=$(grep -o "captured one: [0-9]*" gpurun_out/r2_plain_cfg5ev.log | grep -o "[0-9]*$")
ncu --set full --clock-control none --import-source on -k regex:damf_event_kernel -s ${SK:-10} -c 1 -f \
    -o gpurun_out/r2_evk_cfg5 python tools/prof_r2.py cfg5ev > gpurun_out/r2_ncu_cfg5ev.log 2>&1; echo "ncu evk rc $?"
# cfg-2 split kernels (factor kernel + per-event push kernel)
python tools/prof_r2.py cfg2ev > gpurun_out/r2_plain_cfg2ev.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'damf_event_kernel|damf_ppr_kernel' -s 410 -c 2 -f \
    -o gpurun_out/r2_cfg2_split python tools/prof_r2.py cfg2ev > gpurun_out/r2_ncu_cfg2ev.log 2>&1; echo "ncu cfg2 rc $?"
# whole-GPU push after 1,000 insertions (config-4 shape): launch list with DRAM bytes
PROF_PUSH_ONLY=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r2_ppr_push_launches.csv python tools/prof_ppr.py 23 128 \
    > gpurun_out/r2_ncu_ppr_push.log 2>&1; echo "ncu push rc $?"
ls -la gpurun_out | tail -20
