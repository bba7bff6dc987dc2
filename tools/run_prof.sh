# run tools/configs_bench.py with the profiling build swapped in (experiments only)
cp paper_1608_08648_b200/libovs.so /tmp/libovs_main.so
cp tools/variants/libovs_prof.so paper_1608_08648_b200/libovs.so
python tools/configs_bench.py 3 "$1"
cp /tmp/libovs_main.so paper_1608_08648_b200/libovs.so
