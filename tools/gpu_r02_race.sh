#!/bin/bash
# the single-tile hd-80 causal case that failed a numerics assertion under racecheck
T='tests/test_attention_gpu.py::test_attention_matches_fp32[ql10-kl10-4-2-80-True-128]'
for i in 1 2; do
  timeout 300 compute-sanitizer --tool racecheck python -m pytest "$T" -q 2>&1 | grep -E "passed|failed|Error:|RACECHECK|assert" | head -4
done
timeout 300 compute-sanitizer --tool synccheck python -m pytest "$T" -q 2>&1 | grep -E "passed|failed|ERROR|SUMMARY" | head -4
timeout 300 compute-sanitizer --tool initcheck python -m pytest "$T" -q 2>&1 | grep -E "passed|failed|ERROR|SUMMARY" | head -6
for i in 1 2 3; do timeout 120 python -m pytest "$T" -q 2>&1 | tail -1; done
EMM_ATT_DYN=0 timeout 300 compute-sanitizer --tool racecheck python -m pytest "$T" -q 2>&1 | grep -E "passed|failed" | head -2
