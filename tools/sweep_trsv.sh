#!/bin/bash
# Sweep the trisolve grid caps and poll back-off on the B200 (tools/prof_exact.py).
for b in 1 2 4; do
  for ns in 128 512 2048; do
    echo "solve blocks_per_sm=$b sleep_ns=$ns: $(SAIT_TRSV_BLOCKS_PER_SM=$b SAIT_TRSV_SLEEP_NS=$ns timeout 120 python tools/prof_exact.py 128 2>&1 | grep -E 'exact ilu' | tr -s ' ')"
  done
done
for ab in 0 4; do
  for ans in 1024 4096; do
    echo "analysis blocks_per_sm=$ab sleep_ns=$ans: $(SAIT_TRSV_ANALYSIS_BLOCKS_PER_SM=$ab SAIT_TRSV_ANALYSIS_SLEEP_NS=$ans timeout 120 python tools/prof_exact.py 128 2>&1 | grep -E 'L only' | tr -s ' ')"
  done
done
