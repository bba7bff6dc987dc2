#!/bin/bash
# Round evidence on one B200 (run under gpurun): bench line, BASELINE configs, emulated ranks, strings,
# then the ncu launch list of one bench step and a full ncu capture of the three level-0 hot kernels.
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench exit $?" >> gpurun_out/${TAG}_bench.err
timeout 600 python tools/configs_bench.py 5 > gpurun_out/${TAG}_configs.jsonl 2>&1
OVS_BENCH_MERGE=1 timeout 300 python tools/configs_bench.py 5 C2-uniform,C2-few,C4 >> gpurun_out/${TAG}_configs.jsonl 2>&1
timeout 900 python tools/dist_virtual_bench.py 1 2 4 8 > gpurun_out/${TAG}_dist_virtual.jsonl 2>&1
timeout 300 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 bash tools/ncu_hot.sh ${TAG}_full
ls -la gpurun_out | tail -20
