#!/bin/bash
# round-2 final evidence on one B200: GPU tests, smoke(), the default bench line,
# the reference arm, and C5 at its true shape
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_final.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.txt 2>&1
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err
timeout 2400 python bench.py --config c5 --warmup 1 --steps 1 --no-cpu-e2e --no-decode \
  > gpurun_out/bench_c5_final.json 2> gpurun_out/bench_c5_final.err
cat gpurun_out/pytest_final.txt; tail -2 gpurun_out/smoke_final.txt
for f in bench_final bench_ref_final bench_c5_final; do
  python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().splitlines()[-1]);print('$f', d.get('value'), d.get('unit'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), d.get('step_frac_of_bf16_sustained'))"
done
