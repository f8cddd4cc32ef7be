"""Scheduler host loop on the C++ library.

Drop-in replacements for the reference's per-pass scheduler helpers, same
names, arguments and results, backed by csrc/host_sched.cpp:

  LoadEstimator          balancer.py:115-164  (read twice per group on every
                         scheduler pass by Scheduler._rebalance_idle,
                         engine.py:964-972: ~70 % of simulator CPU)
  assign_idle_instances  balancer.py:67-84
  place_reservations     partition.py:169-184
  allocate_prefill       partition.py:187-290

Every decision is bit-exact with the reference's Python (tests/
test_sched_port.py fuzzes each function against it and replays the golden
runs with all four installed).  `install(partition_module, balancer_module)`
rebinds them the same way `engine.install` rebinds UnifiedCache.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

import sys

from ._lib import check, lib

# the reference's sum() over floats: Neumaier-compensated on CPython >= 3.12,
# plain left-to-right before (pkg/pyproject.toml declares requires-python >= 3.10)
check(lib.emm_sched_set_float_sum(1 if sys.version_info >= (3, 12) else 0))

_p = lambda a: a.ctypes.data if a.size else None  # noqa: E731


def _cost_vec(profile) -> np.ndarray:
    """The 8 CostProfile fields of emm.h's EMM_COST_* order."""
    return np.array([profile.prefill_rate, profile.parallel_alpha, profile.migration_bandwidth,
                     profile.decode_base, profile.decode_batch_coeff, profile.decode_kv_coeff,
                     profile.encode_rate, profile.decode_batch_threshold], np.float64)


class LoadEstimator:
    """balancer.LoadEstimator on the C++ estimator (balancer.py:115-164)."""

    def __init__(self, profile, window_seconds: float = 60.0, bucket_seconds: float = 5.0):
        self.profile = profile
        self.window = window_seconds
        self.bucket = bucket_seconds
        self._cost = _cost_vec(profile)
        h = C.c_void_p()
        check(lib.emm_estimator_create(self._cost.ctypes.data, float(window_seconds),
                                       float(bucket_seconds), C.byref(h)))
        self._h = h
        self._a, self._pk = C.c_int64(), C.c_int64()
        self._a_ref, self._pk_ref = C.byref(self._a), C.byref(self._pk)
        self._observe = lib.emm_estimator_observe
        self._required = lib.emm_estimator_required
        self._peak = lib.emm_estimator_peak_required
        self._peak_now = None  # peak computed with the last avg_required(now)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib.emm_estimator_destroy(h)
            except Exception:  # interpreter shutdown: the library may be gone
                pass
            self._h = None

    def service_seconds(self, input_tokens: int, image_tokens: int, output_tokens: int) -> float:
        out = C.c_double()
        check(lib.emm_estimator_service_seconds(self._h, int(input_tokens), int(image_tokens),
                                                int(output_tokens), C.byref(out)))
        return out.value

    def observe(self, now: float, input_tokens: int, image_tokens: int,
                output_tokens: int) -> None:
        self._peak_now = None
        check(self._observe(self._h, float(now), int(input_tokens), int(image_tokens),
                            int(output_tokens)))

    def avg_required(self, now: float) -> int:
        # one call computes avg then peak at `now` (both drop the same old
        # events first); peak_required(now) right after reuses it
        rc = self._required(self._h, float(now), self._a_ref, self._pk_ref)
        if rc:
            self._peak_now = None
            check(rc)
        self._peak_now = now
        return self._a.value

    def peak_required(self, now: float) -> int:
        if now == self._peak_now:
            return self._pk.value
        rc = self._peak(self._h, float(now), self._pk_ref)
        if rc:
            check(rc)
        return self._pk.value

    def __len__(self) -> int:
        n = C.c_int64()
        check(lib.emm_estimator_len(self._h, C.byref(n)))
        return n.value


def assign_idle_instances(avg_required: dict, busy_counts: dict,
                          idle_instance_ids: list) -> dict:
    """balancer.py:67-84: group id -> idle instances to receive."""
    gids = list(avg_required)
    n = len(gids)
    if not n:
        return {}
    arr = C.c_int64 * n
    grants = arr()
    check(lib.emm_assign_idle(arr(*gids), arr(*avg_required.values()),
                              arr(*[busy_counts.get(k, 0) for k in gids]), n,
                              len(idle_instance_ids), grants))
    return dict(zip(gids, grants))


def place_reservations(requests: list, headroom: dict) -> dict | None:
    """partition.py:169-184: best-fit packing; None when a request fits nowhere."""
    n = len(requests)
    r = np.array([(s.request_id, s.kv_need) for s in requests], np.int64).reshape(n, 2)
    h = np.array(list(headroom.items()), np.int64).reshape(len(headroom), 2)
    out = np.zeros(max(n, 1), np.int64)
    ok = C.c_int32()
    check(lib.emm_place_reservations(_p(r), n, _p(h), len(headroom), out.ctypes.data,
                                     C.byref(ok)))
    if not ok.value:
        return None
    return {s.request_id: int(i) for s, i in zip(requests, out[:n])}


@dataclass
class PrefillAllocation:
    """partition.PrefillAllocation (partition.py:158-166), same fields."""
    instance_ids: list = field(default_factory=list)
    placements: dict | None = field(default_factory=dict)
    preempted: list = field(default_factory=list)
    forced_preempted: list = field(default_factory=list)
    dropped: list = field(default_factory=list)
    decisions: list = field(default_factory=list)


def allocate_prefill(profile, requests, idle, decode_victims, decode_batch, penalty_w: float,
                     max_instances: int | None = None, extra_homes=None) -> PrefillAllocation:
    """partition.py:187-290 on the C++ allocator: same instance grants,
    placements, forced / opportunistic preemptions, drops and decision log."""
    n_req, n_idle, n_vic = len(requests), len(idle), len(decode_victims)
    extra = extra_homes or []
    req = np.array([(s.request_id, s.kv_need, s.input_len, s.prefill_tokens) for s in requests],
                   np.int64).reshape(n_req, 4)
    idl = np.array([(s.instance_id, s.kv_headroom) for s in idle], np.int64).reshape(n_idle, 2)
    vic = np.array([(v.instance_id, v.kv_unused, v.kv_used, v.capacity, int(bool(v.migratable)))
                    for v in decode_victims], np.int64).reshape(n_vic, 5)
    ext = np.array([(s.instance_id, s.kv_headroom) for s in extra], np.int64).reshape(len(extra),
                                                                                    2)
    outs = np.array(decode_batch.output_lens, np.int64)
    cost = _cost_vec(profile)
    counts = np.zeros(6, np.int64)
    ids = np.zeros(n_idle + n_vic + 1, np.int64)
    place = np.zeros(2 * n_req + 2, np.int64)
    pre = np.zeros(n_vic + 1, np.int64)
    forced = np.zeros(n_vic + 1, np.int64)
    dropped = np.zeros(n_req + 1, np.int64)
    d_inst = np.zeros(n_vic + 1, np.int64)
    d_forced = np.zeros(n_vic + 1, np.int32)
    d_gain = np.zeros(n_vic + 1, np.float64)
    d_cost = np.zeros(n_vic + 1, np.float64)
    check(lib.emm_allocate_prefill(
        cost.ctypes.data, float(penalty_w), -1 if max_instances is None else int(max_instances),
        _p(req), n_req, _p(idl), n_idle, _p(vic), n_vic, _p(outs), len(outs),
        int(decode_batch.remaining_output), int(decode_batch.resident_kv),
        int(decode_batch.n_instances), _p(ext), len(extra), counts.ctypes.data, ids.ctypes.data,
        place.ctypes.data, pre.ctypes.data, forced.ctypes.data, dropped.ctypes.data,
        d_inst.ctypes.data, d_forced.ctypes.data, d_gain.ctypes.data, d_cost.ctypes.data))
    n_ids, n_place, n_pre, n_forced, n_drop, n_dec = (int(c) for c in counts)
    alloc = PrefillAllocation()
    alloc.instance_ids = [int(x) for x in ids[:n_ids]]
    alloc.placements = None if n_place < 0 else {
        int(place[2 * i]): int(place[2 * i + 1]) for i in range(n_place)}
    alloc.preempted = [int(x) for x in pre[:n_pre]]
    alloc.forced_preempted = [int(x) for x in forced[:n_forced]]
    alloc.dropped = [int(x) for x in dropped[:n_drop]]
    alloc.decisions = [{"kind": "preempt_for_prefill", "instance": int(d_inst[i]),
                        "forced": bool(d_forced[i]),
                        "gain": None if math.isnan(d_gain[i]) else float(d_gain[i]),
                        "cost": float(d_cost[i])} for i in range(n_dec)]
    return alloc


_NAMES = {"balancer": ("LoadEstimator", "assign_idle_instances"),
          "partition": ("place_reservations", "allocate_prefill")}


def install(partition_module, balancer_module) -> dict:
    """Rebind the reference's scheduler helpers to the C++ ones (the engine
    resolves them as module attributes: engine.py:23-24, 921-924, 977,
    1073, 1104).  Returns what uninstall() needs."""
    prev = {}
    for mod, names in ((balancer_module, _NAMES["balancer"]),
                       (partition_module, _NAMES["partition"])):
        for name in names:
            prev[(mod, name)] = getattr(mod, name)
            setattr(mod, name, globals()[name])
    return prev


def uninstall(prev: dict) -> None:
    for (mod, name), fn in prev.items():
        setattr(mod, name, fn)
