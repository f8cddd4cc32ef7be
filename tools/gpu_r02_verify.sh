#!/bin/bash
# the committed build end to end: GPU tests, smoke(), the default bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_verify.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_verify.txt 2>&1
timeout 1200 python bench.py > gpurun_out/bench_verify.json 2> gpurun_out/bench_verify.err
cat gpurun_out/pytest_verify.txt; tail -2 gpurun_out/smoke_verify.txt
python -c "import json;d=json.loads(open('gpurun_out/bench_verify.json').read().splitlines()[-1]);print(d.get('value'), (d.get('e2e') or {}).get('value'), d.get('clocks'), (d.get('roofline') or {}).get('frac'))"
