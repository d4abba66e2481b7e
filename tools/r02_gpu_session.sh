set -x
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench_rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err; echo ref_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-plugin-e2e --no-check --e2e-steps 1 > gpurun_out/r02_ncu_list.log 2>&1; echo list_rc=$?
bash tools/ncu_capture.sh r02_p2 "k_seg_prod_p2" 0 -- python bench.py --steps 1 --warmup 0 --no-cpu --no-plugin-e2e --no-check --e2e-steps 1
bash tools/ncu_capture.sh r02_nd "k_seg_prod_nd" 0 -- python bench.py --steps 1 --warmup 0 --no-cpu --no-plugin-e2e --no-check --e2e-steps 1
bash tools/ncu_capture.sh r02_p2pow "k_p2_pow" 1 -- python bench.py --steps 1 --warmup 0 --no-cpu --no-plugin-e2e --no-check --e2e-steps 1
ls -la gpurun_out/
