#!/bin/bash
mkdir -p gpurun_out
( for d in 0 2 4 6; do echo "== EMM_SKINNY_DBG=$d"; EMM_SKINNY_DBG=$d timeout 120 python tools/skinny_prof.py 40 3584 3584 | tail -11;
  EMM_SKINNY_CLUSTER=0 EMM_SKINNY_DBG=$d timeout 120 python tools/skinny_prof.py 40 3584 3584 | tail -11; done ) 2>&1 | tee gpurun_out/skinny_prof3.txt
