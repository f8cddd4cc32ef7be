#!/bin/bash
mkdir -p gpurun_out
( for shp in "64 4608 3584" "64 3584 3584" "64 3584 18944" "64 37888 3584 glu"; do
    timeout 120 python tools/skinny_prof.py $shp 2>&1 | tail -17 | head -9
  done ) > gpurun_out/skinny_phase.txt 2>&1
