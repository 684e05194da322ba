"""Device groups (include/atc_b200.h, atc_group_*): several GPUs of one process.

SURVEY.md §8(e): the unpruned binding space shards naturally — an enumerated
range is cut into contiguous pieces (atc_plan_shards), each device evaluates its
pieces against its own replica of the recorded test sets, and the per-device
results are combined (MIN of the first passing index — the candidate the
reference's rank-order loop, pipeline.cpp:248-310, reaches first —, SUM of the
reason histograms, ordered union of the passing lists).  The reference's caller
is the worker pool of pipeline.cpp:340-355; `Group.member(i)` hands each worker a
context of its own.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib


def plan_shards(counts: Sequence[int], world: int) -> list:
    """atc_plan_shards: [[(begin, end) of job j] for rank r] (host arithmetic)."""
    n = len(counts)
    cnt = np.ascontiguousarray(counts, dtype=np.uint64)
    b = np.zeros(max(world * n, 1), dtype=np.uint64)
    e = np.zeros(max(world * n, 1), dtype=np.uint64)
    rc = _lib.lib().atc_plan_shards(cnt.ctypes.data, n, world, b.ctypes.data, e.ctypes.data)
    if rc != _lib.ATC_OK:
        raise _lib.AtcError(rc, "atc_plan_shards: bad arguments")
    return [[(int(b[r * n + j]), int(e[r * n + j])) for j in range(n)] for r in range(world)]


class _Member(_lib.Context):
    """A group member's context (owned by the group, never destroyed here)."""

    def __init__(self, handle, device: int):  # noqa: D401 - no atc_create
        self.handle, self.device = handle, device

    def close(self) -> None:
        self.handle = None


class Group:
    """atc_group: one context per listed device (a device may repeat)."""

    def __init__(self, devices: Optional[Sequence[int]] = None):
        L = _lib.lib()
        if devices is None:
            self.handle = L.atc_group_create(None, 0)
        else:
            arr = (C.c_int32 * len(devices))(*devices)
            self.handle = L.atc_group_create(arr, len(devices))
        if not self.handle:
            raise _lib.AtcError(_lib.ATC_ERR_DEVICE, "atc_group_create returned NULL")
        err = L.atc_group_last_error(self.handle)
        if err:
            msg = err.decode()
            L.atc_group_destroy(self.handle)
            self.handle = None
            raise _lib.AtcError(_lib.ATC_ERR_DEVICE, msg)
        self.devices = list(devices) if devices is not None else list(range(self.size))

    @property
    def size(self) -> int:
        return int(_lib.lib().atc_group_size(self.handle))

    def member(self, i: int) -> _lib.Context:
        return _Member(_lib.lib().atc_group_member(self.handle, i), self.devices[i])

    def _check(self, rc: int) -> None:
        if rc != _lib.ATC_OK:
            raise _lib.AtcError(rc, _lib.lib().atc_group_last_error(self.handle).decode())

    def upload(self, ts, needed_only: bool = True) -> "GroupTestsets":
        """atc_group_testsets_upload_seeded: the recorded test sets on every member."""
        s, keep = ts.seeded_struct(needed_only)
        out = C.c_void_p()
        self._check(_lib.lib().atc_group_testsets_upload_seeded(self.handle, C.byref(s), C.byref(out)))
        return GroupTestsets(self, out.value, keep)

    def eval_enumerated_many(self, items: list, cap: int = 1 << 16, mode: int = _lib.MODE_FP64) -> list:
        """[(passing indices ascending (<= cap), passing count, reason histogram, first
        passing index or -1)] per (spec, ts, space, begin, end) item."""
        return GroupSweep(self, items, cap, mode, prepared=False).run()

    def sweep(self, items: list, cap: int = 1 << 16, mode: int = _lib.MODE_FP64) -> "GroupSweep":
        return GroupSweep(self, items, cap, mode, prepared=True)

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.lib().atc_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GroupTestsets:
    def __init__(self, group: Group, value, keep):
        self.group, self.value, self.keep = group, value, keep

    def free(self) -> None:
        if self.value and self.group.handle:
            _lib.lib().atc_group_testsets_free(self.group.handle, self.value)
        self.value = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class GroupSweep:
    """atc_group_eval_enumerated_many (one-shot) or atc_group_batch_* (prepared)."""

    def __init__(self, group: Group, items: list, cap: int, mode: int, prepared: bool):
        self.group, self.cap, self.mode, self.n = group, cap, mode, len(items)
        self.jobs = (_lib.GroupJob * max(self.n, 1))()
        self._keep = []
        uploaded = {}
        for j, (spec, ts, space, begin, end) in enumerate(items):
            h = uploaded.get(id(ts))
            if h is None:
                h = uploaded[id(ts)] = group.upload(ts)
            desc = spec.to_desc()
            perms = np.ascontiguousarray(space.perms, dtype=np.uint8)
            surv = np.zeros(max(cap, 1), dtype=np.uint64)
            self._keep.append((desc, perms, surv, h))
            jb = self.jobs[j]
            jb.spec = C.cast(C.pointer(desc), C.c_void_p)
            jb.ts = h.value
            jb.perms = perms.ctypes.data
            jb.n_perms = int(perms.shape[0])
            jb.begin, jb.end = int(begin), int(space.count if end is None else end)
            jb.survivors = surv.ctypes.data
            jb.cap = cap
        self._out = _lib.out_view(self.jobs, self.n, ["n_survivors", "reason_counts", "status", "first_pass"])
        self.handle = None
        if prepared:
            L = _lib.lib()
            self.handle = L.atc_group_batch_create(group.handle, self.jobs, self.n, mode)
            if not self.handle:
                raise _lib.AtcError(_lib.ATC_ERR_ARG, L.atc_group_last_error(group.handle).decode())

    def run(self) -> list:
        L = _lib.lib()
        if self.handle:
            self.group._check(L.atc_group_batch_run(self.group.handle, self.handle))
        else:
            self.group._check(L.atc_group_eval_enumerated_many(self.group.handle, self.jobs, self.n, self.mode))
        o = self._out
        if o["status"].any():
            j = int(np.flatnonzero(o["status"])[0])
            raise _lib.AtcError(int(o["status"][j]), f"job {j}: atc error {int(o['status'][j])}")
        ks = o["n_survivors"].tolist()  # (slices past a buffer's cap end at the cap)
        return list(zip([kp[2][:k].copy() for kp, k in zip(self._keep, ks)], ks, list(o["reason_counts"].copy()),
                        o["first_pass"].tolist()))

    def close(self) -> None:
        if self.handle and self.group.handle:
            _lib.lib().atc_group_batch_destroy(self.group.handle, self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
