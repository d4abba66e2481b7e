# round-2 final measurement session (after the decrypt lane rule and wave-sized encrypt chunks)
set -x
python -m pytest tests -q -m gpu --durations=10 > gpurun_out/f2_tests.log 2>&1; echo tests_rc=$?
python __graft_entry__.py smoke > gpurun_out/f2_smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f2_ref.json 2> gpurun_out/f2_ref.err; echo ref_rc=$?
python tools/train_timing.py tests/configs/vertical_c2_2048.ini 2048 7 4 > gpurun_out/f2_c2_timing.json 2> gpurun_out/f2_c2_timing.err; echo c2_rc=$?
echo done
