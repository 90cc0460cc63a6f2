"""Config-5 input generator (workloads/mc5.py): the host side of the
counter-based recipe K4 implements on the device. Input generation only --
these tests check that the traces are valid wire-format traces and that the
recipe behaves as documented. No GPU."""
import ctypes

import numpy as np
import pytest

import paper_2510_21048_b200 as xm
from workloads import mc5


def test_templates_have_dense_ids():
    for k in (0, 57, len(mc5.TEMPLATES) - 1):
        fixed, per, tag, nids = mc5.template(k)
        ids = tag & 0x0FFFFFFF
        assert ids.max() + 1 == nids
        live, peak = set(), 0
        for j in range(len(ids)):
            if fixed[j] + per[j] > 0:
                assert ids[j] not in live
                live.add(int(ids[j]))
                peak = max(peak, len(live))
            else:
                live.remove(int(ids[j]))
        assert not live                        # closed
        assert peak == nids                    # LIFO recycling: id space == max live


def test_generated_traces_pass_the_loader():
    b = mc5.batch(np.arange(0, 400_000, 997))
    tr = xm.load_traces(b.bytes, b.tag, b.off)        # validation (ids, sizes, closure)
    assert tr.n_traces == b.n_traces and tr.n_events == b.n_events


def test_descriptors_are_per_index():
    d_all = mc5.describe(np.arange(5000))
    idx = np.array([17, 4999, 3, 2500])
    d = mc5.describe(idx)
    for k in ("tpl", "b", "capacity", "seed"):
        assert (d[k] == d_all[k][idx]).all()
    d = mc5.describe(np.arange(200_000))
    assert len(np.unique(d["tpl"])) == len(mc5.TEMPLATES)        # every template drawn
    assert set(np.unique(d["capacity"]).tolist()) == {8 << 30, 12 << 30}


def test_swap_rule():
    k = mc5.TEMPLATES.index(("gpt2", "adamw", "pos0"))
    fixed, per, tag, _ = mc5.template(k)
    by, tg = mc5.instantiate(k, 25, np.uint64(12345))
    ref = fixed + per * 25
    moved = np.flatnonzero(by != ref)
    # swaps are adjacent transpositions of events with different ids
    c = mc5.swap_source(len(fixed), np.uint64(12345))
    keep = c & ~np.r_[False, c[:-1]]
    ids = tag & 0x0FFFFFFF
    keep[:-1] &= ids[:-1] != ids[1:]
    ks = np.flatnonzero(keep)
    assert 0.005 < len(ks) / len(fixed) < 0.03
    assert not (np.diff(ks) == 1).any()
    assert (tg[ks] == tag[ks + 1]).all() and (tg[ks + 1] == tag[ks]).all()
    assert set(moved.tolist()) <= set(ks.tolist()) | set((ks + 1).tolist())


def test_expand_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    t = xm._Tpl(None, None, None, None, 1)
    rc = xm.lib().xm_expand_templates(ctypes.byref(t), None, None, None, 0, None, 1,
                                      None, None, None, None)
    assert rc != 0


def test_c_recipe_equals_numpy_recipe():
    """workloads/mc5gen.c (used for parity on all 1M config-5 traces) builds
    exactly the traces of the documented numpy recipe."""
    idx = np.r_[np.arange(0, 1_000_000, 2011), np.arange(999_000, 999_050)]
    a = mc5.batch(idx)
    b = mc5.batch_fast(idx)
    assert (a.off == b.off).all() and (a.capacity == b.capacity).all()
    assert (a.bytes == b.bytes).all() and (a.tag == b.tag).all()
    # the swap rule fired (the recipe is not the identity)
    fixed, per, tag, tpl_off, _ = mc5.template_pool()
    assert any((b.tag[b.off[t]:b.off[t + 1]] != tag[tpl_off[k]:tpl_off[k + 1]]).any()
               for t, k in enumerate(mc5.describe(idx)["tpl"][:50]))
