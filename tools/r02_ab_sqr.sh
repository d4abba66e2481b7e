#!/bin/bash
# A/B of the TPI=1 Montgomery squaring variants on encrypt/decrypt at 2048 bits
# (base = shipped build; sqr_p2 = digit squarings only; sqr_pow = mod-p
# exponentiation squarings only; sqr = both), interleaved, two rounds.
for r in 1 2; do
  for v in base sqr_p2 sqr_pow sqr; do
    lib=paper_2504_03909_b200/lib/libsfxb_cuda.so
    [ $v != base ] && lib=lib_variants/$v/libsfxb_cuda.so
    SFXB_LIB=$lib python tools/microbench.py --bits 2048 --sizes 262144 1048576 --ops enc dec \
      | sed "s/^{/{\"variant\": \"$v\", \"round\": $r, /" >> gpurun_out/ab_sqr.jsonl
  done
done
