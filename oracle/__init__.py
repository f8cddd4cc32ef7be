"""oracle/ — TEST INFRASTRUCTURE, not product code.

CPU restatements of the reference's algorithms for the hot path, used only as
the parity checker by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs:

  cache_oracle.py   pure-Python restatement of mmsim.cache decisions
                    (pinned against the reference's recorded call logs)
  hash_oracle.c     C restatement of the block-hash / pixel-digest definitions
  hashes.py         ctypes loader of hash_oracle.c (oracle/_build/liboracle.so)
  model_ref.py      fp32 torch restatement of the ViT encoder and the prefill
                    decoder (numerics oracle; the reference has no numerics,
                    SURVEY.md §0, so numeric parity is builder-pinned)
  gen_golden.py     writes tests/golden/* from the reference (build container
                    only; /root/reference does not exist on the GPU box)

The product path (paper_2507_10069_b200) never imports this package.
"""
