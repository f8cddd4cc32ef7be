"""K6 over NCCL point-to-point: grouped ncclSend / ncclRecv between the GPUs
of one process (the transport PAPER.md:316 names for KV migration: NCCL group
P2P on dedicated streams), for execute_migration (pkg/src/mmsim/engine.py:
753-788) and the prefill -> home KV hand-off (SURVEY.md §8e exchange 1).

NCCL is the library doing the transfer (NVLink / NVSwitch P2P between the
devices); this module is its binding: one communicator per physical device
from ncclCommInitAll, and every (layer, K/V) plane of every moving request
sent as one ncclSend / ncclRecv pair inside ONE ncclGroupStart / End, on the
source / destination devices' current streams.  The destination stream also
waits for the source stream, so an event recorded on it after `move_many`
brackets the whole transfer.  Requests whose source and destination are the
same physical device (logical GPUs sharing a B200) use the K6 kernel.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_NCCL_UINT8 = 1


def _find_nccl() -> str:
    try:
        import nvidia.nccl as nn   # the copy torch itself loads
        for p in nn.__path__:
            cand = os.path.join(p, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                return cand
    except Exception:
        pass
    return "libnccl.so.2"


class NcclP2P:
    """Communicators over `devices` (distinct physical CUDA device indices)."""

    def __init__(self, devices):
        devs = sorted({int(d) for d in devices})
        self.devices = devs
        self.rank = {d: i for i, d in enumerate(devs)}
        self.lib = C.CDLL(_find_nccl(), mode=C.RTLD_GLOBAL)
        L = self.lib
        L.ncclGetErrorString.restype = C.c_char_p
        L.ncclCommInitAll.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_int)]
        for fn in (L.ncclSend, L.ncclRecv):
            fn.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        self.comms = (C.c_void_p * len(devs))()
        arr = (C.c_int * len(devs))(*devs)
        self._check(L.ncclCommInitAll(self.comms, len(devs), arr), "ncclCommInitAll")

    def _check(self, rc: int, what: str) -> None:
        if rc != 0:
            raise RuntimeError(f"{what}: NCCL error {rc}: "
                               f"{self.lib.ncclGetErrorString(rc).decode()}")

    def close(self) -> None:
        if getattr(self, "comms", None) is not None:
            for c in self.comms:
                if c:
                    self.lib.ncclCommDestroy(C.c_void_p(c))
            self.comms = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _planes(kv: torch.Tensor, n_rows: int):
        """(pointer, bytes) of rows [0, n_rows) of every (layer, K/V) plane."""
        assert kv.dim() == 4 and kv.stride(3) == 1 and kv.stride(2) == kv.shape[3]
        nbytes = n_rows * kv.shape[3] * kv.element_size()
        out = []
        for li in range(kv.shape[0]):
            for h in range(kv.shape[1]):
                out.append((kv[li, h].data_ptr(), nbytes))
        return out

    def move_many(self, pairs) -> None:
        """pairs: (src [L, 2, rows, d], dst same shape, n_rows) on devices in
        `devices`; all transfers in one NCCL group (src and dst on the same
        device is NCCL's send-to-self, used by the one-GPU tests)."""
        if not pairs:
            return
        L = self.lib
        src_streams, dst_streams = {}, {}
        for src, dst, _ in pairs:
            src_streams[src.device.index] = torch.cuda.current_stream(src.device)
            dst_streams[dst.device.index] = torch.cuda.current_stream(dst.device)
        self._check(L.ncclGroupStart(), "ncclGroupStart")
        try:
            for src, dst, n in pairs:
                a, b = src.device.index, dst.device.index
                ca, cb = self.comms[self.rank[a]], self.comms[self.rank[b]]
                sa, sb = src_streams[a].cuda_stream, dst_streams[b].cuda_stream
                for (ps, nb), (pd, nd) in zip(self._planes(src, n), self._planes(dst, n)):
                    assert nb == nd
                    self._check(L.ncclSend(C.c_void_p(ps), nb, _NCCL_UINT8, self.rank[b],
                                           C.c_void_p(ca), C.c_void_p(sa)), "ncclSend")
                    self._check(L.ncclRecv(C.c_void_p(pd), nd, _NCCL_UINT8, self.rank[a],
                                           C.c_void_p(cb), C.c_void_p(sb)), "ncclRecv")
        finally:
            self._check(L.ncclGroupEnd(), "ncclGroupEnd")
        # destination streams also wait for the sending streams
        for dv, ds in dst_streams.items():
            for sv, ss in src_streams.items():
                if sv != dv:
                    ev = torch.cuda.Event()
                    ev.record(ss)
                    ds.wait_event(ev)
