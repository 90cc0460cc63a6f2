"""Seeded synthetic trace generators shared by tests, bench and smoke.

This module is deliberately *method-free*: it produces raw alloc/free event
traces in the wire format and nothing else. It contains none of the
allocator arithmetic (no 512 B rounding, no pool or segment sizing, no
best-fit) -- that lives independently in ``oracle/`` (test infrastructure)
and in ``paper_2510_21048_b200/csrc`` (the product). Neither of those is
imported here, and this module imports neither of them.

Wire format (one batch of T traces, E events):

* ``bytes``    int64[E]   signed request bytes: +req at an alloc, -req at the
                          matching free (the profiler's signed-bytes
                          convention, SPEC.md:27 ``MemArgs``).
* ``tag``      uint32[E]  block id in bits 0-27, stream in bits 28-31.
* ``off``      int64[T+1] trace t owns events [off[t], off[t+1]).
* ``capacity`` uint64[T]  per-trace device capacity (UINT64_MAX = unlimited).

Array order is the replay order (reading Q6).
"""
from .trace import Batch, TraceBuilder, concat, UNLIMITED
from . import rng, fuzz, hand, models, suites

__all__ = ["Batch", "TraceBuilder", "concat", "UNLIMITED",
           "rng", "fuzz", "hand", "models", "suites"]
