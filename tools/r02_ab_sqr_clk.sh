#!/bin/bash
# Clocks / power / throttle reasons sampled while encrypt runs at 1M (base vs sqr_p2)
for v in base sqr_p2 base sqr_p2; do
  lib=paper_2504_03909_b200/lib/libsfxb_cuda.so
  [ $v != base ] && lib=lib_variants/$v/libsfxb_cuda.so
  nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/clk_$v.csv &
  smi=$!
  SFXB_LIB=$lib python tools/microbench.py --bits 2048 --sizes 1048576 4194304 --ops enc \
    | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/ab_sqr_clk.jsonl
  kill $smi
  echo "== $v" >> gpurun_out/clk_all.csv; cat gpurun_out/clk_$v.csv >> gpurun_out/clk_all.csv
done
