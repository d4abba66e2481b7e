# round-2 session 8: full GPU suite, smoke, bench, launch list, 3072-bit C4 rows
set -x
python -m pytest tests -q -m gpu --durations=15 > gpurun_out/s8_tests.log 2>&1; echo tests_rc=$?
python __graft_entry__.py smoke > gpurun_out/s8_smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/s8_bench.json 2> gpurun_out/s8_bench.err; echo bench_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s8_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-plugin-e2e --no-check --e2e-steps 1 > gpurun_out/s8_ncu_list.log 2>&1; echo list_rc=$?
python tools/microbench.py --bits 3072 > gpurun_out/s8_micro3072.jsonl 2> gpurun_out/s8_micro3072.err; echo micro_rc=$?
echo done
