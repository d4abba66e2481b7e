# round-2 session 7: when the offline phase may run (between calls / always / except during decrypt)
set -x
for r in 1 2; do
  for m in between always nodecrypt; do
    SFXB_ENC_PRECOMPUTE=$m LD_PRELOAD=$PWD/paper_2504_03909_b200/lib/libsfxb_cuda_plugin.so oracle/_ref/plugin_bench 1000000 14 256 6 2048 2 4 > gpurun_out/s7_pb_${m}_$r.json 2>&1
  done
done
python tools/train_timing.py tests/configs/vertical_c2_2048.ini 2048 7 4 > gpurun_out/s7_c2_timing.json 2> gpurun_out/s7_c2_timing.err; echo c2_rc=$?
echo done
