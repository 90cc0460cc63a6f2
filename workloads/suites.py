"""The five BASELINE.json configs as seeded synthetic batches.

configs[0] single synthetic trace: 3-layer MLP, 1 iteration, ~500 events, batch 32
configs[1] ResNet-50 training-iteration traces, batch 8..256 step 8 (32 traces)
configs[2] BERT-base / GPT-2 small, AdamW, b=5..55 step 5, zero_grad POS0/POS1,
           3 streams (compute / data loader / optimizer foreach) -> 44 traces
configs[3] 25-model suite x 5209 runs: the first 3903 cells of the ANOVA grid
            + 1306 Monte Carlo draws
configs[4] Monte Carlo: N perturbed traces (1M in the paper-scale run), trace i
           a pure function of (i, salt) so every rank can build its own shard.

Input shapes are a reading (the paper does not state them): CNN inputs are
3x32x32 in the ANOVA/MC suites (batch 200-700 must straddle a 12 GB device,
PAPER.md:373), 3x224x224 in config 2; transformer sequences are 512 tokens.
"""
from __future__ import annotations

import itertools
from typing import List, Tuple

import numpy as np

from . import models as M
from .rng import generator, trace_seed
from .trace import Batch, UNLIMITED

GiB = 1 << 30

CNN_OPTS = ["sgd", "adam", "adamw", "rmsprop", "adagrad"]
TR_OPTS = ["sgd", "adafactor", "adam", "adamw"]
RQ5_OPTS = ["sgd", "adafactor"]
IMG_SUITE = 32
SEQ_SUITE = 512


def _assemble(items: List[Tuple[str, np.ndarray, np.ndarray, int]]) -> Batch:
    names = [it[0] for it in items]
    lens = [len(it[1]) for it in items]
    off = np.zeros(len(items) + 1, np.int64)
    off[1:] = np.cumsum(lens)
    by = np.concatenate([it[1] for it in items]) if items else np.zeros(0, np.int64)
    tg = np.concatenate([it[2] for it in items]) if items else np.zeros(0, np.uint32)
    cap = np.array([it[3] for it in items], np.uint64)
    return Batch(by, tg, off, cap, names)


def config1() -> Batch:
    tpl = M.template("mlp3", "adam", "pos1", iterations=1, micro=20)
    by, tg = M.instantiate(tpl, 32)
    return _assemble([("mlp3/adam/pos1/b32", by, tg, int(UNLIMITED))])


def config2() -> Batch:
    tpl = M.template("resnet50", "sgd_momentum", "pos1", img=224)
    return _assemble([(f"resnet50/sgd_momentum/pos1/b{b}", *M.instantiate(tpl, b), int(UNLIMITED))
                      for b in range(8, 257, 8)])


def config3() -> Batch:
    items = []
    for name in ("bert_base", "gpt2"):
        for zg in ("pos0", "pos1"):
            tpl = M.template(name, "adamw", zg, streams=True, seq=512)
            for b in range(5, 56, 5):
                items.append((f"{name}/adamw/{zg}/b{b}/streams3", *M.instantiate(tpl, b),
                              int(UNLIMITED)))
    return _assemble(items)


def _family(name):
    if name in M.CNNS_PAPER:
        return "cnn"
    if name in M.SMALL_LLMS:
        return "llm"
    if name in M.RQ5:
        return "rq5"
    return "tr"


def _batches(fam):
    return {"cnn": list(range(200, 701, 100)), "tr": list(range(5, 56, 5)),
            "llm": list(range(1, 9)), "rq5": [1]}[fam]


def _opts(fam):
    return {"cnn": CNN_OPTS, "tr": TR_OPTS, "llm": TR_OPTS, "rq5": RQ5_OPTS}[fam]


def anova_cells() -> List[Tuple[str, str, int, int]]:
    """(model, optimizer, batch, repeat) in a fixed order: 3910 cells."""
    cells = []
    for name in M.CNNS_PAPER + M.TRANSFORMERS + M.SMALL_LLMS + M.RQ5:
        fam = _family(name)
        for opt, b, rep in itertools.product(_opts(fam), _batches(fam), range(5)):
            cells.append((name, opt, b, rep))
    return cells


MC_MODELS = M.CNNS_PAPER + M.TRANSFORMERS + M.SMALL_LLMS    # the 22 RQ1-RQ4 models


def mc_draw(i: int, salt: int = 5):
    """Monte Carlo configuration i: model, optimizer, batch,
    zero_grad placement and target GPU (12 GiB RTX 3060 / 8 GiB RTX 4060)."""
    g = generator(trace_seed(i, salt))
    name = MC_MODELS[int(g.integers(0, len(MC_MODELS)))]
    fam = _family(name)
    opts, bs = _opts(fam), _batches(fam)
    opt = opts[int(g.integers(0, len(opts)))]
    b = bs[int(g.integers(0, len(bs)))]
    zg = ("pos0", "pos1")[int(g.integers(0, 2))]
    cap = (12 * GiB, 8 * GiB)[int(g.integers(0, 2))]
    return name, opt, b, zg, cap, g


def _tpl(name, opt, zg):
    return M.template(name, opt, zg, img=IMG_SUITE, seq=SEQ_SUITE)


def anova_trace(k: int, cell):
    name, opt, b, rep = cell
    g = generator(trace_seed(k, 4))
    by, tg = M.instantiate(_tpl(name, opt, "pos1"), b, g, swap_p=0.02)
    return (f"{name}/{opt}/pos1/b{b}/r{rep}", by, tg, int(UNLIMITED))


def mc_trace(i: int, salt: int = 5):
    name, opt, b, zg, cap, g = mc_draw(i, salt)
    by, tg = M.instantiate(_tpl(name, opt, zg), b, g, swap_p=0.02)
    return (f"mc{i}:{name}/{opt}/{zg}/b{b}/cap{cap >> 30}G", by, tg, cap)


def config4(n_anova: int = 3903, n_mc: int = 1306) -> Batch:
    cells = anova_cells()[:n_anova]
    items = [anova_trace(k, c) for k, c in enumerate(cells)]
    items += [mc_trace(i) for i in range(n_mc)]
    return _assemble(items)


def config5(indices, salt: int = 6) -> Batch:
    """Monte Carlo traces with the given global indices (a rank's shard)."""
    return _assemble([mc_trace(int(i), salt) for i in indices])


def mc_lengths(indices, salt: int = 6) -> np.ndarray:
    """Event counts of MC traces without materialising them (for shard planning)."""
    out = np.zeros(len(indices), np.int64)
    for k, i in enumerate(indices):
        name, opt, b, zg, cap, _ = mc_draw(int(i), salt)
        out[k] = len(_tpl(name, opt, zg)[0])
    return out


CONFIGS = {"cfg1": config1, "cfg2": config2, "cfg3": config3, "cfg4": config4}


# ---- the bench's global trace pool -------------------
# index i <  5209: config 4 (ANOVA cells then MC draws with salt 5)
# index i >= 5209: further MC draws (salt 6) -- N GPUs replay N*5209 traces.
N_CFG4 = 5209
N_ANOVA = 3903


def _cell_len(cell):
    name, opt, b, rep = cell
    return len(_tpl(name, opt, "pos1")[0])


def pool_lengths(n: int) -> np.ndarray:
    cells = anova_cells()[:N_ANOVA]
    out = np.zeros(n, np.int64)
    for i in range(n):
        if i < N_ANOVA:
            out[i] = _cell_len(cells[i])
        elif i < N_CFG4:
            name, opt, b, zg, cap, _ = mc_draw(i - N_ANOVA, 5)
            out[i] = len(_tpl(name, opt, zg)[0])
        else:
            name, opt, b, zg, cap, _ = mc_draw(i - N_CFG4, 6)
            out[i] = len(_tpl(name, opt, zg)[0])
    return out


def pool_batch(indices) -> Batch:
    cells = anova_cells()[:N_ANOVA]
    items = []
    for i in indices:
        i = int(i)
        if i < N_ANOVA:
            items.append(anova_trace(i, cells[i]))
        elif i < N_CFG4:
            items.append(mc_trace(i - N_ANOVA, 5))
        else:
            items.append(mc_trace(i - N_CFG4, 6))
    return _assemble(items)
