"""Drop-in integration with the reference scheduler (mmsim.engine).

`install()` rebinds the name `UnifiedCache` that the reference drivers
instantiate per modality group (pkg/src/mmsim/engine.py:932-934, 1449,
1565-1567) to GpuUnifiedCache, so the unchanged scheduler makes every cache
call into the C++ control plane.  `B200Engine` subclasses the reference
Engine and overrides only the stage entry points named in SURVEY.md §8b:

  start_encode    (engine.py:565)  -> ViT encode of the missed images (K1, K4)
  start_prefill   (engine.py:602)  -> K1/K2 match, K3 gather, prefill (K5)
  _handle_prefill_done (engine.py:634) -> brackets the reference's own
                     insert_prefix calls with the KV-scatter registration
  unified_sequence (engine.py:448) -> same symbols, keys precomputed
and, for the coupled driver, its private encode unit (engine.py:1619-1641),
which calls profile.encode_time directly.

Modes:
  "A"  parity: durations stay the reference's analytic ones, so the event
       order - and every cache decision - equals a plain reference run,
       while the real GPU work executes at each hook;
  "B"  measurement: the measured device seconds of each encode / prefill
       job become that job's event duration (TTFT = simulated queueing +
       measured compute).
The duration substitution is a one-shot CostProfile proxy scoped to the
hook, so partition / balancer estimates keep the analytic model
(partition.py:86-131, balancer.py:130-138).
"""
from __future__ import annotations

import contextlib
import ctypes
import math

import torch

from .cache import GpuUnifiedCache
from .keys import SymbolSeq, request_keys

try:
    import mmsim.engine as _E  # type: ignore
except Exception:  # pragma: no cover - reference not installed
    _E = None


def _require():
    if _E is None:
        raise ImportError("mmsim (the reference scheduler) is not importable; install it into "
                          "baseline/_ref or put /root/reference/pkg/src on sys.path")
    return _E


def install(module=None):
    """Make the reference drivers build GpuUnifiedCache; returns the previous
    binding for uninstall()."""
    E = module or _require()
    prev = E.UnifiedCache
    if not (isinstance(prev, type) and issubclass(prev, GpuUnifiedCache)):
        E.UnifiedCache = GpuUnifiedCache
    return prev


def uninstall(prev, module=None):
    E = module or _require()
    E.UnifiedCache = prev


@contextlib.contextmanager
def installed(module=None):
    prev = install(module)
    try:
        yield
    finally:
        uninstall(prev, module)


class _ProfileProxy:
    """CostProfile view with some methods replaced (the timing seam)."""

    def __init__(self, base, **overrides):
        object.__setattr__(self, "_base", base)
        object.__setattr__(self, "_over", overrides)

    def __getattr__(self, name):
        over = object.__getattribute__(self, "_over")
        if name in over:
            return over[name]
        return getattr(object.__getattribute__(self, "_base"), name)


def _timed(fn):
    """Run fn() on the current stream, return (result, device seconds)."""
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    out = fn()
    e.record()
    e.synchronize()
    return out, s.elapsed_time(e) / 1e3


EngineBase = _E.Engine if _E is not None else object


class B200Engine(EngineBase):
    def __init__(self, trace, policy, profile, config=None, slo_input=math.inf, seed=0,
                 hotpath=None, mode: str = "A"):
        E = _require()
        if mode not in ("A", "B"):
            raise ValueError("mode must be 'A' (parity) or 'B' (measured durations)")
        self.hp = hotpath
        self.mode = mode
        self.gpu = {"encode_jobs": 0, "encode_s": 0.0, "prefill_batches": 0, "prefill_s": 0.0,
                    "first_tokens": {}, "device_matched_kv": {}, "host_cached_prefix": {}}
        self._batch_kv: dict = {}
        # request id -> (device index, KV tensor [L, 2, tokens, kv_dim]) resident on
        # its home instance after prefill (the KV the ledger accounts for)
        self.resident: dict = {}
        self.migration_log: list = []
        self.n_gpus = max(1, torch.cuda.device_count()) if hotpath is not None else 1
        with installed(E):
            super().__init__(trace, policy, profile, config, slo_input, seed)
        self._devices = {}
        if self.hp is not None and self.n_gpus > 1:
            from . import _lib
            _lib.declare_more({"emm_enable_peer_access": (ctypes.c_int, [ctypes.c_int,
                                                                         ctypes.c_int])})
            for d in range(self.n_gpus):
                for p in range(self.n_gpus):
                    if d != p:
                        _lib.check(_lib.lib.emm_enable_peer_access(d, p))
        if self.hp is not None:
            for gid, cache in sorted(self.caches.items()):
                self._devices[gid] = self.hp.attach(cache)
            if isinstance(self.driver, E._CoupledDriver):
                orig = self.driver._start_encode_unit

                def coupled_encode(iid, rid, _orig=orig):
                    st = self.requests[rid]
                    with self._encode_seam(st.group_id):
                        return _orig(iid, rid)
                self.driver._start_encode_unit = coupled_encode

    # -------------------------------------------------------------- helpers
    def _device_for(self, group_id):
        cd = self._devices.get(group_id)
        if cd is None and self.hp is not None:
            cd = self.hp.cd  # cache disabled: a private, never-populated index
        return cd

    @contextlib.contextmanager
    def _encode_seam(self, group_id):
        if self.hp is None:
            yield
            return
        base = self.profile

        def encode_time(missed_images, n_instances):
            cd = self._device_for(group_id)
            _, secs = _timed(lambda: self.hp.encode(list(missed_images), self.now, cd=cd))
            self.gpu["encode_jobs"] += 1
            self.gpu["encode_s"] += secs
            if self.mode == "B":
                return secs
            return base.encode_time(missed_images, n_instances)

        self.profile = _ProfileProxy(base, encode_time=encode_time)
        try:
            yield
        finally:
            self.profile = base

    # ---------------------------------------------------------- overridden
    def unified_sequence(self, req):
        """engine.py:448-461, with the symbol keys precomputed (vectorised)."""
        symbols, weights = super().unified_sequence(req)
        codec = None
        for c in self.caches.values():
            codec = getattr(c, "codec", None)
            break
        if codec is None:
            return symbols, weights
        k, w = request_keys(codec, req)
        seq = SymbolSeq(k, w, symbols)
        return seq, seq.weights

    def start_encode(self, st, instance_ids, missed_images):
        with self._encode_seam(st.group_id):
            return super().start_encode(st, instance_ids, missed_images)

    def start_prefill(self, group, specs, instance_ids, placements, migration_wait,
                      compute_width=None):
        if self.hp is None:
            return super().start_prefill(group, specs, instance_ids, placements,
                                         migration_wait, compute_width)
        cd = self._device_for(group.id)
        states = [self.requests[s.request_id] for s in specs]
        reqs = [st.req for st in states]
        cached = [st.cached_prefix for st in states]
        res, secs = _timed(lambda: self.hp.prefill(reqs, cached, cd=cd))
        self.gpu["prefill_batches"] += 1
        self.gpu["prefill_s"] += secs
        ids = res.next_ids.cpu().tolist()
        mkv = res.matched_kv.cpu().tolist()
        for st, tok, m, c in zip(states, ids, mkv, cached):
            self.gpu["first_tokens"][st.req.id] = tok
            self.gpu["device_matched_kv"][st.req.id] = m
            self.gpu["host_cached_prefix"][st.req.id] = c
        base = self.profile
        if self.mode == "B":
            self.profile = _ProfileProxy(base, prefill_time=lambda tokens, width: secs)
        try:
            batch = super().start_prefill(group, specs, instance_ids, placements,
                                          migration_wait, compute_width)
        finally:
            self.profile = base
        self._batch_kv[batch.batch_id] = (res.kv, cd)
        return batch

    def device_of(self, instance_id: int) -> int:
        """Instance i runs on GPU i mod n_gpus."""
        return instance_id % self.n_gpus

    def _handle_prefill_done(self, ev):
        entry = self._batch_kv.pop(ev.payload.get("batch"), None)
        batch = self.batches.get(ev.payload.get("batch"))
        live = (entry is not None and batch is not None and not batch.finished
                and ev.payload.get("gen") == batch.gen)
        if live and self.cache_for(batch.group_id) is not None:
            self.hp.prepare_insert(entry[0], cd=entry[1])
        try:
            super()._handle_prefill_done(ev)
        finally:
            if live:
                self.hp.finish_insert(cd=entry[1])
                bkv = entry[0]
                for r, rid in enumerate(bkv.rids):
                    n = self.requests[rid].req.total_input_len
                    row0 = int(bkv.row0[r])
                    home = self.requests[rid].home_instance
                    self.resident[rid] = (self.device_of(home),
                                          bkv.req_kv[:, :, row0:row0 + n])
            elif entry is not None and batch is not None and not batch.finished:
                self._batch_kv[ev.payload.get("batch")] = entry  # stale event: keep

    def _complete_request(self, st):
        self.resident.pop(st.req.id, None)
        return super()._complete_request(st)

    def execute_migration(self, src, moves, after, reason):
        """engine.py:753-788: move every resident's KV from `src` to its planned
        destination with K6 (TMA-bulk row copy; peer-to-peer over NVLink when
        the instances live on different GPUs).  Mode B charges the measured
        copy time instead of migration_cost(kv_used) (costmodel.py:138-142)."""
        if self.hp is None:
            return super().execute_migration(src, moves, after, reason)
        from . import dataplane
        todo = [(rid, dst) for rid, dst in sorted(moves.items()) if rid in self.resident]
        moved_bytes = 0

        def copy_all():
            nonlocal moved_bytes
            for rid, dst in todo:
                dev_src, kv = self.resident[rid]
                dev_dst = self.device_of(dst)
                with torch.cuda.device(dev_dst):
                    out = torch.empty(kv.shape, dtype=kv.dtype, device=f"cuda:{dev_dst}")
                    dataplane.kv_copy_rows(kv, None, out, None, kv.shape[2])
                self.resident[rid] = (dev_dst, out)
                moved_bytes += kv.numel() * kv.element_size()
        _, secs = _timed(copy_all)
        self.migration_log.append({"src": src, "moves": dict(moves), "rows_moved": len(todo),
                                   "bytes": moved_bytes, "seconds": secs, "reason": reason})
        base = self.profile
        if self.mode == "B":
            self.profile = _ProfileProxy(base, migration_cost=lambda kv_used: secs)
        try:
            return super().execute_migration(src, moves, after, reason)
        finally:
            self.profile = base


def run(trace, policy, profile, config=None, slo_input=math.inf, seed=0, hotpath=None,
        mode="A"):
    """B200 counterpart of mmsim.engine.run (engine.py:1718-1722)."""
    return B200Engine(trace, policy, profile, config, slo_input, seed, hotpath=hotpath,
                      mode=mode).run()
