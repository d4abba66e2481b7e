#!/bin/bash
# A/B of 3072-bit lanes per instance: encrypt step 1 (T1) and the digit exponentiation (TP)
for r in 1 2; do
  for v in base tp48_2 t1_48_1 both48; do
    lib=paper_2504_03909_b200/lib/libsfxb_cuda.so
    [ $v != base ] && lib=lib_variants/$v/libsfxb_cuda.so
    SFXB_LIB=$lib python tools/microbench.py --bits 3072 --sizes 65536 262144 1048576 --ops enc dec \
      | sed "s/^{/{\"variant\": \"$v\", \"round\": $r, /" >> gpurun_out/ab_3072.jsonl
  done
done
