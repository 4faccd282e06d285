"""Integer-nanosecond time base (mirrors batchsym/units.py:1-37).

Every time point and duration on the scheduler path is an int64 tick count
in nanoseconds; configuration in ms/us is converted exactly once.
"""

NS_PER_US = 10**3
NS_PER_MS = 10**6
NS_PER_S = 10**9

#: sentinels kept well inside int64 so tick arithmetic cannot overflow
#: (units.py:16-17); the CUDA engine uses the same values (engine_core.cuh).
TIME_INF = 2**62
NEG_INF = -(2**62)


def _to_ns(value: float, scale: int) -> int:
    # Python's round() is round-half-even on the float product, exactly like
    # the reference's int(round(x * scale)).
    return int(round(value * scale))


def ms_to_ns(ms: float) -> int:
    return _to_ns(ms, NS_PER_MS)


def us_to_ns(us: float) -> int:
    return _to_ns(us, NS_PER_US)


def s_to_ns(s: float) -> int:
    return _to_ns(s, NS_PER_S)


def ns_to_ms(ns: int) -> float:
    return ns / NS_PER_MS


def ns_to_s(ns: int) -> float:
    return ns / NS_PER_S
