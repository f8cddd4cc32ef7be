#!/bin/bash
# session-4 checks: N>1 bench paths on one GPU; NVTX-scoped ncu capture of one stage
mkdir -p gpurun_out
bash tools/gpu_r02_multiproc.sh > gpurun_out/s4_multiproc.txt 2>&1
EMM_NVTX=1 timeout 600 ncu --nvtx --nvtx-include "emm.prefill/" --metrics gpu__time_duration.sum --csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_nvtx_prefill.csv 2> gpurun_out/s4_nvtx.err
echo "nvtx rc=$?" >> gpurun_out/s4_multiproc.txt
