"""Independent brute-force model of the Simulator, used ONLY to pin the oracle.

It shares no code or data structure with oracle/xmo.c: there are no block
objects, no free list, no prev/next links and no merge code. Each live segment
is the sorted list of its *allocated* extents; the free blocks are, by
definition, the gaps between those extents (BFC's coalescing maximality,
SPEC.md:216, makes every free block a maximal gap). Best fit is an exhaustive
minimum over all gaps (PAPER.md:258 (iii); SPEC.md:248 tie order (size, segment,
offset)); a free simply deletes the extent, which merges the neighbouring gaps
by construction. Reclamation deletes segments with no extents (PAPER.md:259-260,
reading Q3). Runs in pure Python: only for traces of a few thousand events.
"""
from __future__ import annotations

import bisect

MiB = 1 << 20
UNLIMITED = (1 << 64) - 1


def rnd(req, g=512, div=0):
    """512 B round-up; with torch's roundup_power2_divisions:div (NEXT-4 variant)
    a request above g*div goes to the next of the div equal steps between the
    powers of two around it (a power of two stays)."""
    if div > 1 and req > g * div:
        lo = 1 << (req.bit_length() - 1)          # 2^k <= req < 2^(k+1)
        if lo == req:
            return req
        steps = [lo + i * (lo // div) for i in range(div + 1)]   # lo ... 2*lo
        return min(x for x in steps if x >= req)
    return max(g, -(-req // g) * g)


def seg_size(s):
    if s <= MiB:
        return 2 * MiB
    if s < 10 * MiB:
        return 20 * MiB
    return -(-s // (2 * MiB)) * (2 * MiB)


def split_ok(small, rem, strict=True):
    if small:
        return rem >= 512
    return rem > MiB if strict else rem >= MiB


class Seg:
    __slots__ = ("base", "size", "stream", "small", "ext")

    def __init__(self, base, size, stream, small):
        self.base, self.size, self.stream, self.small = base, size, stream, small
        self.ext = []  # sorted [(start, end, id)]

    def gaps(self):
        a = self.base
        for (s, e, _) in self.ext:
            if s > a:
                yield (a, s - a)
            a = e
        if a < self.base + self.size:
            yield (a, self.base + self.size - a)


def simulate(bytes_, tag, capacity=UNLIMITED, strict=True, bases=None, div=0, reclaim=0,
             msplit=None, nsr=20 * MiB, gc=0.0):
    """bases: optional segment base addresses in creation order (e.g. the real
    cudaMalloc addresses torch got); default = bump addresses (reading Q4).
    msplit / nsr / gc: torch's max_split_size (bytes), max_non_split_rounding
    and garbage_collection_threshold knobs (NEXT-4, readings Q26/Q27), stated
    here on gaps: a free block's AGE is the number of large-pool searches since
    a gap with exactly its bounds appeared."""
    segs = []
    gc_on = gc > 0.0 and capacity != UNLIMITED
    searches = {False: 0, True: 0}               # per pool (small flag)
    birth = {}                                   # (base, start, len) -> searches then

    def gaps_now():
        return {(g.base, a, L): g for g in segs for (a, L) in g.gaps()}

    def age(g):
        return searches[False] - birth[(g.base, g.base, g.size)]

    def drop(g):
        nonlocal reserved
        segs.remove(g)
        reserved -= g.size
        out["n_seg_release"] += 1
    where = {}     # id -> (seg, start, end, s, request)
    nxt = 0
    reserved = blk = tensor = 0
    out = dict(peak_allocated=0, peak_allocated_idx=0, peak_allocated_blk=0,
               peak_allocated_blk_idx=0, peak_reserved=0, peak_reserved_idx=0,
               n_seg_alloc=0, n_seg_release=0, max_live_segments=0, status=0)
    curve = []
    i = 0
    for i in range(len(bytes_)):
        nb = int(bytes_[i])
        bid = int(tag[i]) & ((1 << 28) - 1)
        st = int(tag[i]) >> 28
        if nb > 0:
            s = rnd(nb, div=div)
            small = s <= MiB
            if gc_on:
                searches[small] += 1
            best = None
            for g in segs:
                if g.stream != st or g.small != small:
                    continue
                for (a, L) in g.gaps():
                    if L >= s and (best is None or (L, a) < (best[0], best[1])):
                        best = (L, a, g)
            if best is not None and msplit is not None:
                # an oversized best fit is refused (and nothing else is tried)
                if (s < msplit and best[0] >= msplit) or (s >= msplit and best[0] >= s + nsr):
                    best = None
            if best is None and gc_on:
                bar = int(gc * float(capacity))
                if reserved > bar:
                    target, got = reserved - bar, 0
                    empty = [g for g in segs if not g.small and not g.ext]
                    ages = sum(age(g) for g in empty)
                    n_ok, freed_any = len(empty), True
                    while empty and got < target and freed_any and n_ok > 0:
                        mean = ages / n_ok
                        old = [g for g in empty if age(g) >= mean]
                        freed_any = bool(old)
                        for g in old:
                            got += g.size
                            ages -= age(g)
                            n_ok -= 1
                            empty.remove(g)
                            drop(g)
            if best is None:
                need = seg_size(s)
                refit = True       # torch: a failed release_available goes straight on
                if reserved + need > capacity and reclaim == 0 and msplit is not None:
                    key = max(s, msplit)
                    mine = [(L, a, g) for g in segs if g.stream == st and g.small == small
                            for (a, L) in g.gaps()]
                    fit = [x for x in mine if x[0] >= key]
                    if fit:
                        L, a, g = min(fit, key=lambda x: (x[0], x[1]))
                        assert not g.ext, "an oversize free block is a whole segment"
                        drop(g)
                    else:
                        got = 0
                        for L, a, g in sorted(mine, key=lambda x: (x[0], x[1]), reverse=True):
                            if got >= key or L < msplit:
                                break
                            assert not g.ext, "an oversize free block is a whole segment"
                            got += L
                            drop(g)
                        refit = got >= key
                if reserved + need > capacity and reclaim == 1:
                    # SPEC.md:283 D3: empty segments, largest first (then lowest
                    # base), only until the request fits
                    for g in sorted([g for g in segs if not g.ext], key=lambda g: (-g.size, g.base)):
                        if reserved + need <= capacity:
                            break
                        segs.remove(g)
                        reserved -= g.size
                        out["n_seg_release"] += 1
                    if reserved + need > capacity:
                        out["status"] = 1
                        break
                elif reserved + need > capacity or not refit:
                    keep = []
                    for g in segs:
                        if g.ext:
                            keep.append(g)
                        else:
                            reserved -= g.size
                            out["n_seg_release"] += 1
                    segs = keep
                    if reserved + need > capacity:
                        out["status"] = 1
                        break
                if bases is not None and out["n_seg_alloc"] < len(bases):
                    g = Seg(bases[out["n_seg_alloc"]], need, st, small)
                else:
                    g = Seg(nxt, need, st, small)
                nxt += need
                segs.append(g)
                reserved += need
                out["n_seg_alloc"] += 1
                out["max_live_segments"] = max(out["max_live_segments"], len(segs))
                best = (need, g.base, g)
            L, a, g = best
            no_split = msplit is not None and not small and s >= msplit
            take = s if split_ok(small, L - s, strict) and not no_split else L
            bisect.insort(g.ext, (a, a + take, bid))
            where[bid] = (g, a, a + take, s)
            blk += take
            tensor += s
        else:
            g, a, e, s = where.pop(bid)
            g.ext.remove((a, e, bid))
            blk -= e - a
            tensor -= s
        if tensor > out["peak_allocated"]:
            out["peak_allocated"], out["peak_allocated_idx"] = tensor, i
        if blk > out["peak_allocated_blk"]:
            out["peak_allocated_blk"], out["peak_allocated_blk_idx"] = blk, i
        if reserved > out["peak_reserved"]:
            out["peak_reserved"], out["peak_reserved_idx"] = reserved, i
        curve.append((tensor, blk, reserved))
        if gc_on:
            now = gaps_now()
            birth = {k: birth.get(k, searches[g.small]) for k, g in now.items()}
    else:
        i = len(bytes_)
    out["events_done"] = i
    out["final_reserved"] = reserved
    out["final_allocated"] = tensor
    out["final_allocated_blk"] = blk
    out["n_free_blocks_end"] = sum(1 for g in segs for _ in g.gaps())
    return out, curve
