# round-2 session 6: passive-party gh conversion in one kernel (k_gh_nd_direct) — parity subset,
# bench, and the offline phase between calls vs always through the plugin (4 trees each, twice)
set -x
python -m pytest tests -q -m gpu -x -k "histogram or e2e or scale or edges or group or dist" > gpurun_out/s6_tests.log 2>&1; echo tests_rc=$?
python bench.py --no-cpu > gpurun_out/s6_bench.json 2> gpurun_out/s6_bench.err; echo bench_rc=$?
SFXB_GH_ND_DIRECT=0 python bench.py --no-cpu --no-plugin-e2e > gpurun_out/s6_bench_twostep.json 2> gpurun_out/s6_bench_twostep.err; echo bench2_rc=$?
for r in 1 2; do
  LD_PRELOAD=$PWD/paper_2504_03909_b200/lib/libsfxb_cuda_plugin.so oracle/_ref/plugin_bench 1000000 14 256 6 2048 2 4 > gpurun_out/s6_pb_default_$r.json 2>&1
  SFXB_ENC_PRECOMPUTE=always LD_PRELOAD=$PWD/paper_2504_03909_b200/lib/libsfxb_cuda_plugin.so oracle/_ref/plugin_bench 1000000 14 256 6 2048 2 4 > gpurun_out/s6_pb_always_$r.json 2>&1
done
echo done
