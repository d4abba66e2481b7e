#!/bin/bash
# A/B of k_p2_pow launch chunking (SFXB_P2_WAVES waves per launch) on encrypt/decrypt at 2048 bits
for r in 1 2; do
  for ch in 0 1 2 4 7; do
    SFXB_P2_WAVES=$ch python tools/microbench.py --bits 2048 --sizes 262144 1048576 4194304 --ops enc dec \
      | sed "s/^{/{\"chunk\": $ch, \"round\": $r, /" >> gpurun_out/ab_chunk.jsonl
  done
done
for v in sqr_p2 sqr; do
  for ch in 1 2; do
    SFXB_LIB=lib_variants/$v/libsfxb_cuda.so SFXB_P2_WAVES=$ch python tools/microbench.py --bits 2048 --sizes 262144 1048576 4194304 --ops enc dec \
      | sed "s/^{/{\"chunk\": \"$v-$ch\", \"round\": 1, /" >> gpurun_out/ab_chunk.jsonl
  done
done
