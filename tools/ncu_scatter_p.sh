#!/bin/bash
# DRAM traffic and time of the level-0 scatter / histogram / bucket sort versus p
for P in 1024 2048 4096; do
  python tools/prof_one.py $P 64 > gpurun_out/sp_plain_$P.log 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum --clock-control none \
      --kernel-name-base demangled -k 'regex:k_(hist|scatter|bucket_sort)<\(int\)0' --csv \
      --log-file gpurun_out/sp_$P.csv python tools/prof_one.py $P 64 > /dev/null 2>&1
done
