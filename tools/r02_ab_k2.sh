# A/B of K2 build variants on the bench (device value), base first and last
set -x
run() { SFXB_LIB=$2 python bench.py --steps 5 --warmup 3 --no-cpu --no-plugin-e2e --no-check --e2e-steps 1 > gpurun_out/ab_$1.json 2> gpurun_out/ab_$1.err; }
run base paper_2504_03909_b200/lib/libsfxb_cuda.so
for v in nd_minb4 nd_pf nd_tpi2 k_tpi2; do [ -f lib_variants/$v/libsfxb_cuda.so ] && run $v lib_variants/$v/libsfxb_cuda.so; done
run base2 paper_2504_03909_b200/lib/libsfxb_cuda.so
echo done
