"""Weak-scaling traces for bench.py --gpus N — TEST/BENCH INFRASTRUCTURE,
runs only in the build container (imports the read-only reference).

The C3 recipe of SURVEY.md §8d at N times the load (qps 1.5 N, same horizon,
seed and multimodal burst; SURVEY §8d "weak scaling optional at qps ∝ n"),
written with the reference's own generator and trace writer
(pkg/src/mmsim/workload.py generate, core.py:277-281 write_trace) and
gzipped: tests/golden/traces/c3_x{N}.jsonl.gz for N = 2..8 (N = 1 is
c3.jsonl).  bench.py shards each over its N ranks with the cache-affine
router (driver.route), so every GPU serves ~1/N of an N-times-larger trace.
"""
import dataclasses
import gzip
import os
import shutil
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gen_golden import GOLDEN, _import_mmsim  # noqa: E402


def main():
    cache, engine, experiments, metrics, workload, core = _import_mmsim()
    share = experiments.resolve_dataset_profile("sharegpt4o-like")
    rep = dataclasses.replace
    for n in range(2, 9):
        tr = workload.generate(
            rep(share, duplicate_image_rate=0.5, duplicate_prefix_rate=0.5), 1.5 * n, 120.0,
            seed=1, bursts=[workload.BurstSpec(40, 30, 3, "multimodal")])
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "t.jsonl")
            core.write_trace(p, tr)
            out = os.path.join(GOLDEN, "traces", f"c3_x{n}.jsonl.gz")
            with open(p, "rb") as fi, gzip.open(out, "wb", compresslevel=9) as fo:
                shutil.copyfileobj(fi, fo)
        print(n, len(tr), sum(r.total_input_len for r in tr))


if __name__ == "__main__":
    main()
