# round-2 measurement session: C4 sweep to 16M, compute-sanitizer, whole C1 runs
python -m pytest tests -q -m gpu -k "encode_batch or group or e2e" > gpurun_out/r02_t3.log 2>&1; echo t3_rc=$?
set -x
compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_smoke.py k512_c0ffee > gpurun_out/r02_racecheck.log 2>&1; echo racecheck_rc=$?
compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_smoke.py k2048_7 > gpurun_out/r02_memcheck.log 2>&1; echo memcheck_rc=$?
compute-sanitizer --tool synccheck python tools/sanitize_smoke.py k512_c0ffee > gpurun_out/r02_synccheck.log 2>&1; echo synccheck_rc=$?
python tools/c1_timing.py > gpurun_out/r02_c1_training.json 2> gpurun_out/r02_c1_training.err; echo c1_rc=$?
python tools/microbench.py > gpurun_out/r02_micro.jsonl 2> gpurun_out/r02_micro.err; echo micro_rc=$?
