# round-2 final measurement session
set -x
python -m pytest tests -q -m gpu --durations=15 > gpurun_out/final_tests.log 2>&1; echo tests_rc=$?
python __graft_entry__.py smoke > gpurun_out/final_smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo ref_rc=$?
python tools/train_timing.py tests/configs/vertical_c2_2048.ini 2048 7 4 > gpurun_out/final_c2_timing.json 2> gpurun_out/final_c2_timing.err; echo c2_rc=$?
echo done
