# run tools/configs_bench.py with the debug-check build swapped in (experiments only)
cp paper_1608_08648_b200/libovs.so /tmp/libovs_main.so
cp tools/variants/libovs_dbg.so paper_1608_08648_b200/libovs.so
python tools/configs_bench.py 1 "$1"
cp /tmp/libovs_main.so paper_1608_08648_b200/libovs.so
