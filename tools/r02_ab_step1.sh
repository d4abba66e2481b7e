#!/bin/bash
# A/B of encrypt step 1 launch chunking (SFXB_STEP1_WAVES) at 1024/2048 bits, interleaved
for r in 1 2; do
  for w in 0 1 2; do
    SFXB_STEP1_WAVES=$w python tools/microbench.py --bits 1024 2048 --sizes 262144 1048576 --ops enc \
      | sed "s/^{/{\"waves1\": $w, \"round\": $r, /" >> gpurun_out/ab_step1.jsonl
  done
done
