# round-2: offline phase between calls vs always vs off; bins handle; squaring off by default
set -x
python -m pytest tests -q -m gpu -x --durations=10 > gpurun_out/t7.log 2>&1; echo tests_rc=$?
python bench.py > gpurun_out/b7.json 2> gpurun_out/b7.err; echo bench_rc=$?
SFXB_ENC_PRECOMPUTE=always LD_PRELOAD=$PWD/paper_2504_03909_b200/lib/libsfxb_cuda_plugin.so oracle/_ref/plugin_bench 1000000 14 256 6 2048 2 4 > gpurun_out/r02_pb_always.json 2>&1
python tools/train_timing.py tests/configs/vertical_c2_2048.ini 2048 7 3 > gpurun_out/r02_c2_timing2.json 2> gpurun_out/r02_c2_timing2.err
echo done
