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
       measured compute), and every decode step lasts the B200 decode step
       measured for its batch and resident KV (decode.DecodeStepModel:
       CUDA-graph replays of real decode steps + the paged decode attention's
       measured seconds per KV byte), replacing decode_step_time.
The duration substitution is a one-shot CostProfile proxy scoped to the
hook, so partition / balancer estimates keep the analytic model
(partition.py:86-131, balancer.py:130-138).
"""
from __future__ import annotations

import contextlib
import math
import os

import torch

from . import dataplane, ops
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
                 hotpath=None, mode: str = "A", native_sched: bool = True,
                 transport: str = "kernel", verify_migration: bool | None = None):
        E = _require()
        # debug mode: every K6 move is checked by an
        # XXH64 checksum of the source and destination rows (dataplane.kv_checksum);
        # a mismatch raises.  Default from EMM_KV_CHECKSUM=1.
        if verify_migration is None:
            verify_migration = os.environ.get("EMM_KV_CHECKSUM", "") == "1"
        self.verify_migration = bool(verify_migration)
        # K6 transport for the KV hand-off and migrations: "kernel" (SM-driven
        # peer row copy) or "copy_engine" (one strided DMA per request)
        if transport not in ("kernel", "copy_engine", "nccl"):
            raise ValueError("transport must be 'kernel', 'copy_engine' or 'nccl'")
        self.transport = transport
        self._nccl = None
        # native_sched: the scheduler's host helpers (load estimator, idle
        # grants, reservation placement, prefill allocation) run on the C++
        # port for the engine's lifetime (sched.py, bit-exact)
        self._native_sched = native_sched
        if mode not in ("A", "B"):
            raise ValueError("mode must be 'A' (parity) or 'B' (measured durations)")
        from .pipeline import HotPathSet
        # one HotPath per logical GPU; instance i runs on GPU i mod n (§8e)
        if hotpath is None:
            self.hps = []
        elif isinstance(hotpath, HotPathSet):
            self.hps = list(hotpath.paths)
        else:
            self.hps = [hotpath]
        self.hp = self.hps[0] if self.hps else None
        self.mode = mode
        self.gpu = {"encode_jobs": 0, "encode_s": 0.0, "prefill_batches": 0, "prefill_s": 0.0,
                    "first_tokens": {}, "device_matched_kv": {}, "host_cached_prefix": {},
                    "encode_split": 0, "prefill_split": 0, "handoffs": 0, "handoff_bytes": 0,
                    "device_of_prefill": {}}
        self._batch_kv: dict = {}
        # request id -> (logical GPU, KV tensor [L, 2, tokens, kv_dim]) resident on
        # its home instance's GPU after prefill (the KV the ledger accounts for)
        self.resident: dict = {}
        self.migration_log: list = []
        self._dmodel = None
        self.gpu["decode_steps_modelled"] = 0
        self.n_gpus = max(1, len(self.hps))
        with installed(E), self._sched_installed(E):
            super().__init__(trace, policy, profile, config, slo_input, seed)
        self._devices = {}
        if self.hp is not None:
            # each modality group's cache (host tree + GPU index + KV pool +
            # image slabs) lives on one GPU; the others reach it peer-to-peer
            for gid, cache in sorted(self.caches.items()):
                self._devices[gid] = self.hps[gid % self.n_gpus].attach(cache)
            if isinstance(self.driver, E._CoupledDriver):
                orig = self.driver._start_encode_unit

                def coupled_encode(iid, rid, _orig=orig):
                    st = self.requests[rid]
                    with self._encode_seam(st.group_id, [iid]):
                        return _orig(iid, rid)
                self.driver._start_encode_unit = coupled_encode
                if self.mode == "B":
                    orig_dec = self.driver._start_decode_unit

                    def coupled_decode(iid, _orig=orig_dec):
                        # engine.py:1688: one instance's batch step, measured model
                        base = self.profile
                        self.profile = _ProfileProxy(
                            base, decode_step_time=lambda b, n, kv: self._decode_step(b, n, kv))
                        try:
                            return _orig(iid)
                        finally:
                            self.profile = base
                    self.driver._start_decode_unit = coupled_decode

    @contextlib.contextmanager
    def _sched_installed(self, E):
        if not self._native_sched:
            yield
            return
        from . import sched
        prev = sched.install(E.part, E.bal)
        try:
            yield
        finally:
            sched.uninstall(prev)

    def run(self):
        with self._sched_installed(_require()):
            return super().run()

    # -------------------------------------------------------------- helpers
    def _uses_nccl(self, src_dev, dst_dev) -> bool:
        """NCCL P2P between distinct physical GPUs; the same device (logical
        GPUs sharing one B200) keeps the K6 kernel."""
        return self.transport == "nccl" and src_dev.index != dst_dev.index

    def _local_transport(self) -> str:
        return "kernel" if self.transport == "nccl" else self.transport

    def _nccl_peers(self):
        if self._nccl is None:
            from .nccl_p2p import NcclP2P
            self._nccl = NcclP2P(sorted({hp.device.index for hp in self.hps}))
        return self._nccl

    def _device_for(self, group_id):
        cd = self._devices.get(group_id)
        if cd is None and self.hp is not None:
            # cache disabled: a private, never-populated index
            if self.hp.cd is None:
                self.hp.new_cache()
            cd = self.hp.cd
        return cd

    def _gpus_of(self, instance_ids) -> list[int]:
        """Distinct logical GPUs of a job's instances, in instance order."""
        out = []
        for i in instance_ids:
            d = self.device_of(i)
            if d not in out:
                out.append(d)
        return out or [0]

    def _encode_on(self, images, instance_ids, cd) -> float:
        """An encode job's missed images split over its instances' GPUs,
        balanced by tokens (data parallel over images, §8e); slabs stay on
        the GPU that encoded them and prefill reads them peer-to-peer.
        Returns the job's device seconds: the slowest GPU's share."""
        from .pipeline import split_balanced
        uniq, seen = [], set()
        for img in images:
            if img.content_hash not in seen and img.content_hash not in cd.slabs:
                seen.add(img.content_hash)
                uniq.append(img)
        gpus = self._gpus_of(instance_ids)
        parts = split_balanced([img.token_count for img in uniq], len(gpus))
        timers = []
        for d, idx in zip(gpus, parts):
            if not idx:
                continue
            hp = self.hps[d]
            with torch.cuda.device(hp.device):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                hp.encode([uniq[i] for i in idx], self.now, cd=cd)
                e.record()
            timers.append((s, e))
        if sum(1 for x in parts if x) > 1:
            self.gpu["encode_split"] += 1
        for _, e in timers:
            e.synchronize()
        return max((s.elapsed_time(e) / 1e3 for s, e in timers), default=0.0)

    @contextlib.contextmanager
    def _encode_seam(self, group_id, instance_ids):
        if self.hp is None:
            yield
            return
        base = self.profile

        def encode_time(missed_images, n_instances):
            cd = self._device_for(group_id)
            secs = self._encode_on(list(missed_images), instance_ids, cd)
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
        with self._encode_seam(st.group_id, instance_ids):
            return super().start_encode(st, instance_ids, missed_images)

    def start_prefill(self, group, specs, instance_ids, placements, migration_wait,
                      compute_width=None):
        if self.hp is None:
            return super().start_prefill(group, specs, instance_ids, placements,
                                         migration_wait, compute_width)
        from .pipeline import split_balanced
        cd = self._device_for(group.id)
        states = [self.requests[s.request_id] for s in specs]
        reqs = [st.req for st in states]
        cached = [st.cached_prefix for st in states]
        # the batch's requests split over its compute GPUs, balanced by the
        # tokens each recomputes; each GPU gathers its cached prefixes from
        # the group's pool and hands a request's KV to its home GPU when the
        # placement differs (§8e exchanges 1 and 2)
        width = compute_width if compute_width is not None else len(instance_ids)
        gpus = self._gpus_of(sorted(instance_ids)[:max(1, width)])
        parts = split_balanced([r.total_input_len - c for r, c in zip(reqs, cached)], len(gpus))
        subs = []
        for d, idx in zip(gpus, parts):
            if not idx:
                continue
            hp = self.hps[d]
            with torch.cuda.device(hp.device):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                res = hp.prefill([reqs[i] for i in idx], [cached[i] for i in idx], cd=cd)
                handoff = {}
                nccl_pairs = []
                hs = torch.cuda.Event(enable_timing=True)
                hs.record()
                bk = res.kv
                for j, i in enumerate(idx):
                    rid = states[i].req.id
                    home = self.device_of(placements[rid])
                    if home == d:
                        continue
                    n, row0 = reqs[i].total_input_len, int(bk.row0[j])
                    src = bk.req_kv[:, :, row0:row0 + n]
                    out = torch.empty(src.shape, dtype=src.dtype, device=self.hps[home].device)
                    if self._uses_nccl(src.device, out.device):
                        nccl_pairs.append((src, out, n))
                    else:
                        dataplane.kv_move(src, out, n, self._local_transport())
                    handoff[rid] = (home, out)
                    self.gpu["handoffs"] += 1
                    self.gpu["handoff_bytes"] += out.numel() * out.element_size()
                if nccl_pairs:
                    self._nccl_peers().move_many(nccl_pairs)
                    for _, out, _ in nccl_pairs:  # this stream waits for the receivers
                        ev = torch.cuda.Event()
                        ev.record(torch.cuda.current_stream(out.device))
                        torch.cuda.current_stream().wait_event(ev)
                e.record()
                handoff_ev = (hs, e) if handoff else None
            subs.append((d, idx, res, handoff, s, e, handoff_ev))
        for sub in subs:
            sub[5].synchronize()
        secs = max(sub[4].elapsed_time(sub[5]) / 1e3 for sub in subs)
        for sub in subs:
            if sub[6] is not None:
                self.gpu["handoff_s"] = (self.gpu.get("handoff_s", 0.0)
                                         + sub[6][0].elapsed_time(sub[6][1]) / 1e3)
        if len(subs) > 1:
            self.gpu["prefill_split"] += 1
        self.gpu["prefill_batches"] += 1
        self.gpu["prefill_s"] += secs
        for d, idx, res, _, _, _, _ in subs:
            ids = res.next_ids.cpu().tolist()
            mkv = res.matched_kv.cpu().tolist()
            for i, tok, m in zip(idx, ids, mkv):
                rid = states[i].req.id
                self.gpu["first_tokens"][rid] = tok
                self.gpu["device_matched_kv"][rid] = m
                self.gpu["host_cached_prefix"][rid] = cached[i]
                self.gpu["device_of_prefill"][rid] = d
        base = self.profile
        if self.mode == "B":
            self.profile = _ProfileProxy(base, prefill_time=lambda tokens, width: secs)
        try:
            batch = super().start_prefill(group, specs, instance_ids, placements,
                                          migration_wait, compute_width)
        finally:
            self.profile = base
        self._batch_kv[batch.batch_id] = ([(sub[0], sub[2].kv) for sub in subs],
                                          {rid: h for sub in subs for rid, h in sub[3].items()},
                                          cd)
        return batch

    # ------------------------------------------------------------ decode
    def _decode_step(self, batch: int, n_instances: int, resident_kv: int) -> float:
        """Measured B200 decode step (decode.DecodeStepModel) for the
        reference's (batch, instances, resident KV) arguments
        (costmodel.py:121-136): each instance runs ceil(batch / n) requests
        over kv / n resident tokens."""
        if self._dmodel is None:
            from .decode import DecodeStepModel
            with torch.cuda.device(self.hp.device):
                self._dmodel = DecodeStepModel(self.hp)
            self.gpu["decode_model"] = self._dmodel.as_dict()
        n = max(1, n_instances)
        share = -(-batch // n)
        self.gpu["decode_steps_modelled"] += 1
        return self._dmodel.step_seconds(share, resident_kv / n)

    def decode_step_seconds(self, group):
        """engine.py:433-439; mode B: the measured step (same arguments)."""
        if self.hp is None or self.mode != "B":
            return super().decode_step_seconds(group)
        pool = self.decode_pool(group)
        active = group.active_decode_count()
        if not pool or active < 1:
            return super().decode_step_seconds(group)   # raises the reference's error
        return self._decode_step(active, len(pool), self.group_decode_resident_kv(group))

    def device_of(self, instance_id: int) -> int:
        """Instance i runs on logical GPU i mod n_gpus."""
        return instance_id % self.n_gpus

    def _handle_prefill_done(self, ev):
        entry = self._batch_kv.pop(ev.payload.get("batch"), None)
        batch = self.batches.get(ev.payload.get("batch"))
        live = (entry is not None and batch is not None and not batch.finished
                and ev.payload.get("gen") == batch.gen)
        if live and self.cache_for(batch.group_id) is not None:
            # one scatter source per sub-batch buffer (peer reads when the
            # sub-batch ran on another GPU than the group's pool)
            self.hp.prepare_insert([bk for _, bk in entry[0]], cd=entry[2])
        try:
            super()._handle_prefill_done(ev)
        finally:
            if live:
                self.hp.finish_insert(cd=entry[2])
                # the scatter reads the sub-batch buffers: done before they go
                torch.cuda.synchronize(entry[2].index.device)
                handoff = entry[1]
                for d, bkv in entry[0]:
                    for r, rid in enumerate(bkv.rids):
                        if rid in handoff:
                            self.resident[rid] = handoff[rid]
                            continue
                        n = self.requests[rid].req.total_input_len
                        row0 = int(bkv.row0[r])
                        self.resident[rid] = (d, bkv.req_kv[:, :, row0:row0 + n])
            elif entry is not None and batch is not None and not batch.finished:
                self._batch_kv[ev.payload.get("batch")] = entry  # stale event: keep

    def _complete_request(self, st):
        self.resident.pop(st.req.id, None)
        return super()._complete_request(st)

    @ops.nvtx_stage("emm.migration")
    def execute_migration(self, src, moves, after, reason):
        """engine.py:753-788: move every resident's KV from `src` to its planned
        destination with K6 (TMA-bulk row copy; peer-to-peer over NVLink when
        the instances live on different GPUs).  Mode B charges the measured
        copy time instead of migration_cost(kv_used) (costmodel.py:138-142)."""
        if self.hp is None:
            return super().execute_migration(src, moves, after, reason)
        todo = [(rid, dst) for rid, dst in sorted(moves.items()) if rid in self.resident]
        moved_bytes = 0
        # Stream-ordered K6: each copy runs on its DESTINATION GPU's stream,
        # after an event recorded on the source GPU's stream (the resident KV
        # is complete there); timing brackets every destination stream used
        # and the old source tensors stay referenced until those streams are
        # done, so the source allocator cannot hand their blocks out while a
        # peer is still reading them.
        marks: dict[int, tuple] = {}
        ready: dict[int, torch.cuda.Event] = {}
        keep = []
        nccl_pairs = []
        sums = []   # verify_migration: (rid, source checksum, destination tensor)
        if self.verify_migration:
            for rid, _dst in todo:
                kv = self.resident[rid][1]
                with torch.cuda.device(kv.device):
                    sums.append([rid, dataplane.kv_checksum(kv, None, kv.shape[2])])
        for rid, dst in todo:
            dev_src, kv = self.resident[rid]
            dev_dst = self.device_of(dst)
            src_dev = kv.device
            if src_dev.index not in ready:
                ev = torch.cuda.Event()
                ev.record(torch.cuda.current_stream(src_dev))
                ready[src_dev.index] = ev
            dst_dev = self.hps[dev_dst].device
            with torch.cuda.device(dst_dev):
                stream = torch.cuda.current_stream(dst_dev)
                if dst_dev.index not in marks:
                    s_ev = torch.cuda.Event(enable_timing=True)
                    s_ev.record(stream)
                    marks[dst_dev.index] = (s_ev, stream)
                if src_dev.index != dst_dev.index:
                    stream.wait_event(ready[src_dev.index])
                out = torch.empty(kv.shape, dtype=kv.dtype, device=dst_dev)
                if self._uses_nccl(src_dev, dst_dev):
                    nccl_pairs.append((kv, out, kv.shape[2]))
                else:
                    dataplane.kv_move(kv, out, kv.shape[2], self._local_transport())
            keep.append(kv)
            self.resident[rid] = (dev_dst, out)
            moved_bytes += kv.numel() * kv.element_size()
        if nccl_pairs:  # one NCCL group for the whole migration
            self._nccl_peers().move_many(nccl_pairs)
        secs = 0.0
        ends = []
        for dev, (s_ev, stream) in marks.items():
            e_ev = torch.cuda.Event(enable_timing=True)
            e_ev.record(stream)
            ends.append((s_ev, e_ev))
        for s_ev, e_ev in ends:
            e_ev.synchronize()
            secs = max(secs, s_ev.elapsed_time(e_ev) / 1e3)
        checked = None
        if sums:   # after the timed region: the destination rows, then compare
            for rec in sums:
                out = self.resident[rec[0]][1]
                with torch.cuda.device(out.device):
                    rec.append(dataplane.kv_checksum(out, None, out.shape[2]))
            for rid, a, b in sums:
                if int(a.item()) != int(b.item()):
                    raise RuntimeError(f"KV migration checksum mismatch for request {rid}: "
                                       f"{int(a.item()) & (2**64 - 1):#x} != "
                                       f"{int(b.item()) & (2**64 - 1):#x}")
            checked = len(sums)
        del keep
        self.gpu["migration_bytes"] = self.gpu.get("migration_bytes", 0) + moved_bytes
        self.gpu["migration_s"] = self.gpu.get("migration_s", 0.0) + secs
        self.migration_log.append({"src": src, "moves": dict(moves), "rows_moved": len(todo),
                                   "bytes": moved_bytes, "seconds": secs, "reason": reason,
                                   "checksums_verified": checked})
        base = self.profile
        if self.mode == "B":
            self.profile = _ProfileProxy(base, migration_cost=lambda kv_used: secs)
        try:
            return super().execute_migration(src, moves, after, reason)
        finally:
            self.profile = base


def run(trace, policy, profile, config=None, slo_input=math.inf, seed=0, hotpath=None,
        mode="A", transport="kernel"):
    """B200 counterpart of mmsim.engine.run (engine.py:1718-1722)."""
    return B200Engine(trace, policy, profile, config, slo_input, seed, hotpath=hotpath,
                      mode=mode, transport=transport).run()
