#!/bin/bash
mkdir -p gpurun_out
( for d in 0 2 8 16; do echo "== DBG $d"; EMM_SKINNY_DBG=$d timeout 120 python tools/skinny_prof.py 40 37888 3584 glu | tail -16 | grep -E "acc_ready|epi_done|c0_|c1_"; done ) 2>&1 | tee gpurun_out/skinny_prof5.txt
