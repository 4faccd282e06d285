"""Canonical digests of scheduler outputs, shared by the fixture generator
(make_golden.py, run against the Python reference) and the tests."""
from __future__ import annotations

import hashlib

import numpy as np

TRACE_KIND = {"dispatch": 0, "drop": 1, "shrink": 2}


def _h(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
        h.update(np.int64(a.size).tobytes())
        h.update(a.tobytes())
    return h.hexdigest()[:32]


def trace_digest(ticks, midx) -> str:
    return _h(ticks, midx)


def requests_digest(dispatch, start, finish, batch, outcome) -> str:
    return _h(dispatch, start, finish, batch, outcome)


def gpu_logs_digest(gpu_logs) -> str:
    flat = []
    for g, log in enumerate(gpu_logs):
        for s, f, m, b in log:
            flat.extend((g, s, f, m, b))
    return _h(flat)


def event_trace_digest(trace) -> str:
    flat = []
    for t, kind, mid, gid, size, start, finish, rids in trace:
        flat.extend((t, TRACE_KIND[kind], mid, gid, size, start, finish, len(rids)))
        flat.extend(rids)
    return _h(flat)


def text_digest(text: str) -> str:
    """Digest of one output file's exact bytes (outputs.py writers)."""
    return hashlib.sha256(text.encode("utf-8")).hexdigest()[:32]
