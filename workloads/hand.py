"""Hand-built traces whose expected results are fixed by the paper, SPEC.md or
closed forms. The traces live here (inputs only); the expected values and
their citations live in ``tests/golden/hand_traces.json``.

Units: MiB = 2**20 B. One stream, unlimited capacity unless stated.
"""
from __future__ import annotations

from typing import Callable, Dict

from .trace import Batch, TraceBuilder

MiB = 1 << 20
KiB = 1 << 10


def _one(fn: Callable[[TraceBuilder], None], capacity=None, name="") -> Batch:
    b = TraceBuilder()
    fn(b)
    b.end_trace(capacity=capacity, name=name)
    return b.build()


def h1(r: int, n: int) -> Batch:
    """H1: n allocs of the same request r <= 1 MiB, no frees."""
    def f(b):
        for i in range(n):
            b.alloc(i, r)
    return _one(f, name=f"H1(r={r},n={n})")


def h2(r: int, n: int) -> Batch:
    """H2: n allocs of r with 1 MiB < round(r) < 10 MiB, no frees."""
    def f(b):
        for i in range(n):
            b.alloc(i, r)
    return _one(f, name=f"H2(r={r},n={n})")


def h3(order: str) -> Batch:
    """H3 (Q11 counterexample): sizes in 512 B units; a small segment is 4096 units."""
    u = 512

    def f(b):
        b.alloc(0, 2048 * u)   # A
        b.alloc(1, 2048 * u)   # D
        if order == "early":
            b.free(0)
            b.alloc(2, 1024 * u)   # B
        else:
            b.alloc(2, 1024 * u)   # B
            b.free(0)
        b.alloc(3, 2048 * u)   # C
        b.alloc(4, 1536 * u)   # E
        b.alloc(5, 1536 * u)   # F
    return _one(f, name=f"H3-{order}")


def h4(order: str) -> Batch:
    """H4: Fig. 2 reconstruction: X=40 MiB live, A=78 MiB, B=78 MiB."""
    def f(b):
        b.alloc(0, 40 * MiB)   # X
        b.alloc(1, 78 * MiB)   # A
        if order == "late":
            b.alloc(2, 78 * MiB)   # B
            b.free(1)
        else:
            b.free(1)
            b.alloc(2, 78 * MiB)
    return _one(f, name=f"H4-{order}")


def h5(two_streams: bool) -> Batch:
    """H5: alloc 1 MiB on stream 0, free, alloc 1 MiB on stream 1 (or 0)."""
    def f(b):
        b.alloc(0, MiB, stream=0)
        b.free(0, stream=0)
        b.alloc(1, MiB, stream=1 if two_streams else 0)
    return _one(f, name=f"H5-{'two' if two_streams else 'one'}")


def h6() -> Batch:
    """H6: one 19 MiB alloc -> 20 MiB segment, remainder exactly 1 MiB."""
    return _one(lambda b: b.alloc(0, 19 * MiB), name="H6")


def h7() -> Batch:
    """H7 = SPEC S:253: capacity 2 MiB; 512 B, free, 2 MiB -> reclaim then OOM."""
    def f(b):
        b.alloc(0, 512)
        b.free(0)
        b.alloc(1, 2 * MiB)
    return _one(f, capacity=2 * MiB, name="H7")


def spec_examples() -> Dict[str, Batch]:
    """SPEC.md allocator_sim worked examples as traces."""
    out = {}
    # S:251 empty state, alloc 512
    out["S251"] = _one(lambda b: b.alloc(0, 512), name="S251")

    # S:252 one Free 1024 in the small pool, alloc 600 -> exact fit, no split.
    # Build the state: [A 1024 | B 1024 | rest]; free A leaves a Free 1024 that is
    # not adjacent to the segment's tail free block.
    def s252(b):
        b.alloc(0, 1024)
        b.alloc(1, 1024)
        b.free(0)
        b.alloc(2, 600)
    out["S252"] = _one(s252, name="S252")
    out["S253"] = h7()

    # S:260 [Used A 512 | Free 512 | Used B 512], free A -> [Free 1024 | Used B 512]
    def s260(b):
        b.alloc(0, 512)     # A
        b.alloc(1, 512)     # hole
        b.alloc(2, 512)     # B
        b.alloc(3, MiB)                # fill the rest of the small segment exactly
        b.alloc(4, MiB - 3 * 512)      # (two small-pool requests; both <= 1 MiB)
        b.free(1)
        b.free(0)
    out["S260"] = _one(s260, name="S260")

    # S:261 free both neighbours of a middle block -> one Free block spanning all three
    def s261(b):
        b.alloc(0, 512)
        b.alloc(1, 512)
        b.alloc(2, 512)
        b.alloc(3, MiB)
        b.alloc(4, MiB - 3 * 512)
        b.free(0)
        b.free(2)
        b.free(1)
    out["S261"] = _one(s261, name="S261")

    # S:262 free the only Used block -> segment fully free, reserved unchanged
    def s262(b):
        b.alloc(0, 4096)
        b.free(0)
    out["S262"] = _one(s262, name="S262")

    # S:269 [Alloc 512, Free] -> curve (512, 2 MiB), (0, 2 MiB)
    def s269(b):
        b.alloc(0, 512)
        b.free(0)
    out["S269"] = _one(s269, name="S269")
    # S:270 empty sequence
    out["S270"] = _one(lambda b: None, name="S270")
    return out


def paper_examples() -> Dict[str, Batch]:
    """P:169 "requesting 2MB for a 1MB tensor"; "a 20MB block for a 10MB tensor"."""
    return {
        "P169": _one(lambda b: b.alloc(0, 1_000_000), name="P169"),
        "P654": _one(lambda b: b.alloc(0, 10_000_000), name="P654"),
        "P654-10MiB": _one(lambda b: b.alloc(0, 10 * MiB), name="P654-10MiB"),
    }


def all_named() -> Dict[str, Batch]:
    d = {}
    d["H1a"] = h1(716_800, 37)
    d["H1b"] = h1(1, 37)
    d["H1c"] = h1(512, 37)
    d["H1d"] = h1(513, 37)
    d["H2a"] = h2(3 * MiB // 2, 23)
    d["H2b"] = h2(13 * MiB // 2, 23)
    d["H3-early"] = h3("early")
    d["H3-late"] = h3("late")
    d["H4-late"] = h4("late")
    d["H4-early"] = h4("early")
    d["H5-two"] = h5(True)
    d["H5-one"] = h5(False)
    d["H6"] = h6()
    d["H7"] = h7()
    d.update(spec_examples())
    d.update(paper_examples())
    return d


def h8() -> Batch:
    """H8 (SPEC.md:283 D3 vs torch release-all): a 2 MiB small and a 20 MiB
    large segment are cached (fully free); a 12 MiB request on another stream
    needs a new segment under a 32 MiB capacity."""
    def f(b):
        b.alloc(0, 512)
        b.alloc(1, 2 * MiB)
        b.free(0)
        b.free(1)
        b.alloc(2, 12 * MiB, stream=1)
        b.free(2, stream=1)
    return _one(f, capacity=32 * MiB, name="H8")
