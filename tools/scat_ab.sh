python tools/phase_bench.py paper_1608_08648_b200/libovs.so tools/vso/libovs_sb16.so tools/vso/libovs_sb16x2.so tools/vso/libovs_sb16x2b0.so
for v in sb16 sb16x2 sb16x2b0; do
  OVS_LIB_PATH=tools/vso/libovs_$v.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_scatter_wc --csv python tools/prof_one.py 2>/dev/null | grep -E "dram|duration" | awk -F'","' -v v=$v '{print v, $(NF-2), $(NF-1), $NF}'
done
