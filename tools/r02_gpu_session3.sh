# round-2: correctness of the squaring + offline phase, A/B of the squaring, steady-state plugin timing
set -x
python -m pytest tests -q -m gpu -x --durations=10 > gpurun_out/t6.log 2>&1; echo tests_rc=$?
python tools/microbench.py --bits 1024 2048 --sizes 262144 1048576 --ops enc dec > gpurun_out/r02_ab_sqr.jsonl 2>&1
SFXB_LIB=$PWD/lib_variants/nosqr/libsfxb_cuda.so python tools/microbench.py --bits 1024 2048 --sizes 262144 1048576 --ops enc dec > gpurun_out/r02_ab_nosqr.jsonl 2>&1
LD_PRELOAD=$PWD/paper_2504_03909_b200/lib/libsfxb_cuda_plugin.so oracle/_ref/plugin_bench 1000000 14 256 6 2048 2 4 > gpurun_out/r02_pb_pre.json 2>&1
SFXB_ENC_PRECOMPUTE=0 LD_PRELOAD=$PWD/paper_2504_03909_b200/lib/libsfxb_cuda_plugin.so oracle/_ref/plugin_bench 1000000 14 256 6 2048 2 4 > gpurun_out/r02_pb_nopre.json 2>&1
python tools/train_timing.py tests/configs/vertical_c2_2048.ini 2048 7 3 > gpurun_out/r02_c2_timing.json 2> gpurun_out/r02_c2_timing.err
echo done
