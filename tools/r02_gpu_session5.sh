# round-2 session 5: one-wave exponentiation launches + digit squarings — bench, launch list,
# ncu of the encrypt exponentiation, C4 sweep, plugin phase profile, configs[1] training timing
set -x
python bench.py > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err; echo bench_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-plugin-e2e --no-check --e2e-steps 1 > gpurun_out/s5_ncu_list.log 2>&1; echo list_rc=$?
bash tools/ncu_capture.sh s5_p2pow "k_p2_pow" 1 -- python bench.py --steps 1 --warmup 0 --no-cpu --no-plugin-e2e --no-check --e2e-steps 1
SFXB_PLUGIN_PROFILE=1 LD_PRELOAD=$PWD/paper_2504_03909_b200/lib/libsfxb_cuda_plugin.so oracle/_ref/plugin_bench 1000000 14 256 6 2048 2 4 > gpurun_out/s5_pb_profile.json 2> gpurun_out/s5_pb_profile.log; echo pb_rc=$?
python tools/train_timing.py tests/configs/vertical_c2_2048.ini 2048 7 4 > gpurun_out/s5_c2_timing.json 2> gpurun_out/s5_c2_timing.err; echo c2_rc=$?
python tools/microbench.py > gpurun_out/s5_micro.jsonl 2> gpurun_out/s5_micro.err; echo micro_rc=$?
echo done
