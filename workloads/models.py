"""Synthetic training-iteration traces shaped like the paper's 25 workloads.

The paper's models (12 CNNs, 10 Transformers, 3 larger
Transformers for RQ5) are described here by approximate public architecture
facts (layer counts, widths, vocabulary, parameter tensors) -- SHAPING ONLY,
not a parity target. A trace is one model, one optimizer, one
zero_grad placement (Fig. 1 POS0/POS1), one batch size b and
3 iterations (PAPER.md:196 footnote), built the way PyTorch's standard loop
 allocates:

  model.to(device): parameters (persistent)              P:241 "Model Parameters"
  per iteration:   [zero_grad POS1] batch data (one iteration)  P:242 "Batch Data"
                   forward: workspace, output, free dead inputs   P:243 "Activations"
                   [zero_grad POS0] backward: grad-ins, param grads,
                   frees of saved activations                     P:244 "Gradients"
                   optimizer.step: persistent state in iteration 1,
                   foreach temporaries every step                 P:245 "Optimizer"
  teardown: every remaining block freed (closed trace, reading Q13)

Every event size is ``fixed + per_sample * b`` bytes (fp32 tensors), so a
template is built once per (model, optimizer, zero_grad, streams) and
instantiated for any batch size with numpy.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache
from typing import Dict, List, Optional, Tuple

import numpy as np

F32 = 4


# ----------------------------------------------------------------------------
# Op graph description
# ----------------------------------------------------------------------------
@dataclass
class Op:
    out: int                       # output numel per sample (0 = in-place / no output)
    params: List[Tuple[int, int]] = field(default_factory=list)  # (rows, cols) per param
    saves_in: bool = False         # input kept for backward
    saves_out: bool = False        # output kept for backward
    extra: List[Tuple[int, int]] = field(default_factory=list)   # saved side tensors (fixed_bytes, per_sample_bytes)
    ws: int = 0                    # forward workspace bytes per sample
    ws_fixed: int = 0              # forward workspace fixed bytes
    res_start: bool = False        # input is also the residual branch
    res_add: bool = False          # adds the pending residual


def _p(n):          # 1-D parameter
    return (n, 1)


def _m(r, c):       # 2-D parameter
    return (r, c)


# ----------------------------- CNN families ---------------------------------
def _conv(cin, cout, k, hw_out, bias=False, ws=True, groups=1):
    ps = [_m(cout, cin // groups * k * k)] + ([_p(cout)] if bias else [])
    return Op(out=cout * hw_out * hw_out, params=ps, saves_in=True,
              ws=(cin * hw_out * hw_out * F32 // 4) if (ws and k > 1) else 0,
              ws_fixed=(1 << 20) if (ws and k > 1) else 0)


def _bn(c, hw):
    return Op(out=c * hw * hw, params=[_p(c), _p(c)], saves_in=True,
              extra=[(c * F32, 0), (c * F32, 0)])


def _act(c, hw, inplace=True):
    # torchvision uses ReLU(inplace=True): no new storage, output saved
    if inplace:
        return Op(out=0, saves_out=False)
    return Op(out=c * hw * hw, saves_out=True)


def vgg(depth: int, img: int = 224) -> List[Op]:
    cfg = {16: [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"],
           19: [64, 64, "M", 128, 128, "M", 256, 256, 256, 256, "M", 512, 512, 512, 512, "M",
                512, 512, 512, 512, "M"]}[depth]
    ops, c, hw = [], 3, img
    for v in cfg:
        if v == "M":
            hw = max(1, hw // 2)
            ops.append(Op(out=c * hw * hw, saves_in=True, extra=[(0, 8 * c * hw * hw)]))  # pool + int64 indices
        else:
            ops.append(_conv(c, v, 3, hw, bias=True))
            ops.append(_act(v, hw))
            c = v
    ops.append(Op(out=c * 7 * 7, saves_in=False))                    # adaptive avgpool
    for (i, o) in ((25088, 4096), (4096, 4096)):
        ops.append(Op(out=o, params=[_m(o, i), _p(o)], saves_in=True))
        ops.append(_act(o, 1))
        ops.append(Op(out=o, saves_out=False, extra=[(0, o)]))       # dropout mask (bool)
    ops.append(Op(out=1000, params=[_m(1000, 4096), _p(1000)], saves_in=True))
    return ops


def resnet(blocks: Tuple[int, int, int, int], img: int = 224) -> List[Op]:
    h2, h4 = max(1, img // 2), max(1, img // 4)
    ops = [_conv(3, 64, 7, h2), _bn(64, h2), _act(64, h2),
           Op(out=64 * h4 * h4, saves_in=True, extra=[(0, 8 * 64 * h4 * h4)])]
    cin, hw = 64, h4
    for si, (n, w) in enumerate(zip(blocks, (64, 128, 256, 512))):
        for bi in range(n):
            hw_o = max(1, hw // 2) if (bi == 0 and si > 0) else hw
            cout = 4 * w
            first = True
            for (ci, co, k, h) in ((cin, w, 1, hw), (w, w, 3, hw_o), (w, cout, 1, hw_o)):
                cv = _conv(ci, co, k, h)
                cv.res_start = first
                first = False
                ops += [cv, _bn(co, h)]
                if co != cout:
                    ops.append(_act(co, h))
            if bi == 0:   # downsample branch
                ops += [_conv(cin, cout, 1, hw_o), _bn(cout, hw_o)]
            ops.append(Op(out=cout * hw_o * hw_o, res_add=True))
            ops.append(_act(cout, hw_o))
            cin, hw = cout, hw_o
    ops.append(Op(out=cin, saves_in=False))
    ops.append(Op(out=1000, params=[_m(1000, cin), _p(1000)], saves_in=True))
    return ops


def inverted_residual_net(stages, stem=32, head=1280, se=False, act_inplace=False,
                          img: int = 224) -> List[Op]:
    """MobileNetV2/V3, MnasNet, RegNet-ish, ConvNeXt-ish generic stage builder.

    stages: list of (expand, cout, n, stride, k)."""
    h2 = max(1, img // 2)
    ops = [_conv(3, stem, 3, h2), _bn(stem, h2), _act(stem, h2, act_inplace)]
    c, hw = stem, h2
    for (t, co, n, s, k) in stages:
        for i in range(n):
            hw_o = max(1, hw // s) if i == 0 else hw
            hidden = c * t
            has_res = i > 0 and co == c
            first = has_res
            if t != 1:
                cv = _conv(c, hidden, 1, hw)
                cv.res_start = first
                first = False
                ops += [cv, _bn(hidden, hw), _act(hidden, hw, act_inplace)]
            dw = _conv(hidden, hidden, k, hw_o, groups=hidden)
            dw.res_start = first
            ops += [dw, _bn(hidden, hw_o), _act(hidden, hw_o, act_inplace)]
            if se:
                sq = max(8, hidden // 4)
                ops += [Op(out=hidden, saves_in=True),
                        Op(out=sq, params=[_m(sq, hidden), _p(sq)], saves_in=True),
                        Op(out=hidden, params=[_m(hidden, sq), _p(hidden)], saves_in=True),
                        Op(out=hidden * hw_o * hw_o, saves_in=True)]
            ops += [_conv(hidden, co, 1, hw_o), _bn(co, hw_o)]
            if has_res:
                ops.append(Op(out=co * hw_o * hw_o, res_add=True))
            c, hw = co, hw_o
    ops += [_conv(c, head, 1, hw), _bn(head, hw), _act(head, hw, act_inplace),
            Op(out=head, saves_in=False),
            Op(out=1000, params=[_m(1000, head), _p(1000)], saves_in=True)]
    return ops


def convnext(depths, dims, img: int = 224) -> List[Op]:
    hw = max(1, img // 4)
    ops = [Op(out=dims[0] * hw * hw, params=[_m(dims[0], 3 * 16), _p(dims[0])], saves_in=True),
           Op(out=dims[0] * hw * hw, params=[_p(dims[0]), _p(dims[0])], saves_in=True,
              extra=[(0, 2 * F32 * hw * hw)])]
    for si, (d, c) in enumerate(zip(depths, dims)):
        if si > 0:
            hw = max(1, hw // 2)
            ops += [Op(out=dims[si - 1] * hw * hw * 4, params=[_p(dims[si - 1]), _p(dims[si - 1])],
                       saves_in=True, extra=[(0, 2 * F32 * hw * hw * 4)]),
                    Op(out=c * hw * hw, params=[_m(c, dims[si - 1] * 4), _p(c)], saves_in=True)]
        for _ in range(d):
            n = hw * hw
            dwc = Op(out=c * n, params=[_m(c, 49), _p(c)], saves_in=True, res_start=True,
                     ws=c * n // 2)
            ops += [dwc,
                    Op(out=c * n, params=[_p(c), _p(c)], saves_in=True, extra=[(0, 2 * F32 * n)]),
                    Op(out=4 * c * n, params=[_m(4 * c, c), _p(4 * c)], saves_in=True),
                    Op(out=4 * c * n, saves_in=True),                                  # GELU
                    Op(out=c * n, params=[_m(c, 4 * c), _p(c)], saves_in=True),
                    Op(out=c * n, params=[_p(c)], saves_in=True),                      # layer scale
                    Op(out=c * n, res_add=True)]
    ops += [Op(out=dims[-1], saves_in=False),
            Op(out=dims[-1], params=[_p(dims[-1]), _p(dims[-1])], saves_in=True),
            Op(out=1000, params=[_m(1000, dims[-1]), _p(1000)], saves_in=True)]
    return ops


# -------------------------- Transformer families ----------------------------
def transformer(L, d, heads, vocab, seq, ffn=None, kv_heads=None, gated=False,
                rms=False, tied=True, bias=True, pos_emb=True, dec_layers=0) -> List[Op]:
    ffn = ffn or 4 * d
    kv_heads = kv_heads or heads
    hd = d // heads
    kvd = kv_heads * hd
    S = seq
    B = (lambda n: [_p(n)] if bias else [])
    ops = [Op(out=S * d, params=[_m(vocab, d)] + ([_m(S, d)] if pos_emb else []), saves_in=True)]

    def norm():
        return Op(out=S * d, params=[_p(d)] if rms else [_p(d), _p(d)], saves_in=True,
                  extra=[(0, S * F32)] if rms else [(0, 2 * S * F32)])

    def layer(cross=False):
        out = []
        n1 = norm()
        n1.res_start = True
        out += [n1,
                Op(out=S * (d + 2 * kvd), params=[_m(d + 2 * kvd, d)] + B(d + 2 * kvd), saves_in=True),
                Op(out=heads * S * S, saves_in=True, ws=heads * S * S * F32 // 8),     # scores
                Op(out=heads * S * S, saves_out=True),                                   # softmax
                Op(out=heads * S * S, extra=[(0, heads * S * S)]),                       # dropout mask
                Op(out=S * d, saves_in=True),                                            # attn @ v
                Op(out=S * d, params=[_m(d, d)] + B(d), saves_in=True),
                Op(out=S * d, res_add=True)]
        if cross:
            n2 = norm()
            n2.res_start = True
            out += [n2, Op(out=S * d, params=[_m(d, d)] + B(d), saves_in=True),
                    Op(out=heads * S * S, saves_out=True),
                    Op(out=S * d, params=[_m(d, d)] + B(d), saves_in=True),
                    Op(out=S * d, res_add=True)]
        n3 = norm()
        n3.res_start = True
        out.append(n3)
        if gated:
            out += [Op(out=2 * S * ffn, params=[_m(2 * ffn, d)], saves_in=True),
                    Op(out=S * ffn, saves_in=True),                                      # silu(gate)*up
                    Op(out=S * d, params=[_m(d, ffn)], saves_in=True)]
        else:
            out += [Op(out=S * ffn, params=[_m(ffn, d)] + B(ffn), saves_in=True),
                    Op(out=S * ffn, saves_in=True),                                      # gelu
                    Op(out=S * d, params=[_m(d, ffn)] + B(d), saves_in=True)]
        out.append(Op(out=S * d, res_add=True))
        return out

    for _ in range(L):
        ops += layer()
    for _ in range(dec_layers):
        ops += layer(cross=True)
    ops.append(norm())
    ops.append(Op(out=S * vocab, params=[] if tied else [_m(vocab, d)], saves_in=True))   # logits
    ops.append(Op(out=S * vocab, saves_out=True))                                          # log_softmax
    return ops


# ----------------------------------------------------------------------------
# Model zoo (Qwen3/Pythia and the RQ5 models P:375, 596-612)
# ----------------------------------------------------------------------------
_MBV2 = [(1, 16, 1, 1, 3), (6, 24, 2, 2, 3), (6, 32, 3, 2, 3), (6, 64, 4, 2, 3),
         (6, 96, 3, 1, 3), (6, 160, 3, 2, 3), (6, 320, 1, 1, 3)]
_MBV3L = [(1, 16, 1, 1, 3), (4, 24, 2, 2, 3), (3, 40, 3, 2, 5), (6, 80, 4, 2, 3),
          (6, 112, 2, 1, 3), (6, 160, 3, 2, 5)]
_MBV3S = [(1, 16, 1, 2, 3), (4, 24, 2, 2, 3), (4, 40, 3, 2, 5), (3, 48, 2, 1, 5), (6, 96, 3, 2, 5)]
_MNAS = [(1, 16, 1, 1, 3), (3, 24, 3, 2, 3), (3, 40, 3, 2, 5), (6, 80, 3, 2, 5),
         (6, 96, 2, 1, 3), (6, 192, 4, 2, 5), (6, 320, 1, 1, 3)]
_REGX = [(1, 32, 1, 2, 3), (1, 64, 2, 2, 3), (1, 160, 7, 2, 3), (1, 400, 12, 2, 3)]
_REGY = [(1, 48, 1, 2, 3), (1, 104, 3, 2, 3), (1, 208, 6, 2, 3), (1, 440, 6, 2, 3)]

# PAPER.md Table 2: 12 CNNs, 10 Transformers (8 + Qwen3-0.6B, Pythia-1b), 3 RQ5 models
CNNS_PAPER = ["vgg16", "vgg19", "resnet101", "resnet152", "mobilenet_v2", "mobilenet_v3_small",
              "mobilenet_v3_large", "mnasnet", "regnet_x_400mf", "regnet_y_400mf",
              "convnext_tiny", "convnext_base"]
TRANSFORMERS = ["distilgpt2", "gpt2", "t5_small", "t5_base", "gpt_neo_125m",
                "opt_125m", "opt_350m", "cerebras_gpt_111m"]
EXTRA = ["resnet50", "bert_base", "mlp3"]   # configs 1-3 only
SMALL_LLMS = ["qwen3_0.6b", "pythia_1b"]
RQ5 = ["llama3.2_3b", "deepseek_r1_qwen_1.5b", "qwen3_4b"]
ALL_MODELS = CNNS_PAPER + TRANSFORMERS + SMALL_LLMS + RQ5 + EXTRA

SEQ = 512
IMG = 224


@lru_cache(maxsize=None)
def model_ops(name: str, img: int = IMG, seq: int = SEQ) -> Tuple[Op, ...]:
    S = seq
    table = {
        "vgg16": lambda: vgg(16, img), "vgg19": lambda: vgg(19, img),
        "resnet50": lambda: resnet((3, 4, 6, 3), img), "resnet101": lambda: resnet((3, 4, 23, 3), img),
        "resnet152": lambda: resnet((3, 8, 36, 3), img),
        "mobilenet_v2": lambda: inverted_residual_net(_MBV2, img=img),
        "mobilenet_v3_small": lambda: inverted_residual_net(_MBV3S, stem=16, head=576, se=True, img=img),
        "mobilenet_v3_large": lambda: inverted_residual_net(_MBV3L, stem=16, head=960, se=True, img=img),
        "mnasnet": lambda: inverted_residual_net(_MNAS, img=img),
        "regnet_x_400mf": lambda: inverted_residual_net(_REGX, head=400, act_inplace=True, img=img),
        "regnet_y_400mf": lambda: inverted_residual_net(_REGY, head=440, se=True, act_inplace=True, img=img),
        "convnext_tiny": lambda: convnext((3, 3, 9, 3), (96, 192, 384, 768), img),
        "convnext_base": lambda: convnext((3, 3, 27, 3), (128, 256, 512, 1024), img),
        "distilgpt2": lambda: transformer(6, 768, 12, 50257, S),
        "gpt2": lambda: transformer(12, 768, 12, 50257, S),
        "bert_base": lambda: transformer(12, 768, 12, 30522, S, tied=True),
        "t5_small": lambda: transformer(6, 512, 8, 32128, S, ffn=2048, rms=True, bias=False,
                                        pos_emb=False, dec_layers=6),
        "t5_base": lambda: transformer(12, 768, 12, 32128, S, ffn=3072, rms=True, bias=False,
                                       pos_emb=False, dec_layers=12),
        "gpt_neo_125m": lambda: transformer(12, 768, 12, 50257, S),
        "opt_125m": lambda: transformer(12, 768, 12, 50272, S),
        "opt_350m": lambda: transformer(24, 1024, 16, 50272, S),
        "cerebras_gpt_111m": lambda: transformer(10, 768, 12, 50257, S),
        "qwen3_0.6b": lambda: transformer(28, 1024, 16, 151936, S, ffn=3072, kv_heads=8,
                                          gated=True, rms=True, bias=False, pos_emb=False),
        "pythia_1b": lambda: transformer(16, 2048, 8, 50304, S, ffn=8192, bias=True,
                                         pos_emb=False, tied=False),
        "llama3.2_3b": lambda: transformer(28, 3072, 24, 128256, S, ffn=8192, kv_heads=8,
                                           gated=True, rms=True, bias=False, pos_emb=False),
        "deepseek_r1_qwen_1.5b": lambda: transformer(28, 1536, 12, 151936, S, ffn=8960,
                                                     kv_heads=2, gated=True, rms=True,
                                                     bias=False, pos_emb=False, tied=False),
        "qwen3_4b": lambda: transformer(36, 2560, 32, 151936, S, ffn=9728, kv_heads=8,
                                        gated=True, rms=True, bias=False, pos_emb=False),
        "mlp3": lambda: [Op(out=1024, params=[_m(1024, 784), _p(1024)], saves_in=True),
                         Op(out=1024, saves_out=True),
                         Op(out=1024, params=[_m(1024, 1024), _p(1024)], saves_in=True),
                         Op(out=1024, saves_out=True),
                         Op(out=10, params=[_m(10, 1024), _p(10)], saves_in=True)],
    }
    return tuple(table[name]())


def is_transformer(name: str) -> bool:
    return name in TRANSFORMERS or name in SMALL_LLMS or name in RQ5 or name == "bert_base"


def input_numel(name: str, img: int = IMG, seq: int = SEQ) -> Tuple[int, int]:
    """(input numel per sample, element bytes) of the batch data."""
    if name == "mlp3":
        return 784, F32
    if is_transformer(name):
        return seq, 8                   # int64 token ids
    return 3 * img * img, F32


OPTIMIZERS = ["sgd", "sgd_momentum", "adam", "adamw", "rmsprop", "adagrad", "adafactor"]


# ----------------------------------------------------------------------------
# Template builder
# ----------------------------------------------------------------------------
class _Tpl:
    def __init__(self):
        self.sign: List[int] = []
        self.fixed: List[int] = []
        self.per: List[int] = []
        self.bid: List[int] = []
        self.stream: List[int] = []
        self.live: Dict[int, Tuple[int, int, int]] = {}
        self.next = 0
        self.marks: List[Tuple[str, int]] = []     # (phase marker, event position)
        self.kinds: List[str] = []                 # per allocation, in order

    def mark(self, name: str):
        """A training-loop phase boundary before the next event (the profiler's
        user_annotation windows)."""
        self.marks.append((name, len(self.sign)))

    def alloc(self, fixed, per=0, stream=0, kind="act") -> int:
        if fixed + per <= 0:
            fixed = 4
        self.kinds.append(kind)
        h = self.next
        self.next += 1
        self.live[h] = (fixed, per, stream)
        self.sign.append(1)
        self.fixed.append(fixed)
        self.per.append(per)
        self.bid.append(h)
        self.stream.append(stream)
        return h

    def free(self, h: Optional[int]):
        if h is None:
            return
        fixed, per, stream = self.live.pop(h)
        self.sign.append(-1)
        self.fixed.append(fixed)
        self.per.append(per)
        self.bid.append(h)
        self.stream.append(stream)

    def arrays(self):
        return (np.asarray(self.sign, np.int64), np.asarray(self.fixed, np.int64),
                np.asarray(self.per, np.int64), np.asarray(self.bid, np.uint32),
                np.asarray(self.stream, np.uint32))


def _opt_state(opt: str, shape: Tuple[int, int]) -> List[int]:
    r, c = shape
    n = r * c
    if opt in ("sgd",):
        return []
    if opt in ("sgd_momentum", "rmsprop", "adagrad"):
        return [n * F32]
    if opt in ("adam", "adamw"):
        return [n * F32, n * F32]
    if opt == "adafactor":
        return [r * F32, c * F32] if c > 1 else [n * F32]
    raise ValueError(opt)


def _opt_temps(opt: str) -> int:
    """param-sized foreach temporaries per step (torch foreach implementations)."""
    return {"sgd": 0, "sgd_momentum": 0, "adam": 1, "adamw": 1, "rmsprop": 1,
            "adagrad": 1, "adafactor": 1}[opt]


@lru_cache(maxsize=None)
def template(name: str, opt: str, zero_grad: str = "pos1", streams: bool = False,
             iterations: int = 3, img: int = IMG, seq: int = SEQ, micro: int = 0):
    """Event template: (sign, fixed, per_sample, id, stream) numpy arrays.

    micro: small autograd temporaries (alloc+free) per op in forward and backward."""
    return _build(name, opt, zero_grad, streams, iterations, img, seq, micro).arrays()


@lru_cache(maxsize=None)
def template_phases(name: str, opt: str, zero_grad: str = "pos1", streams: bool = False,
                    iterations: int = 3, img: int = IMG, seq: int = SEQ, micro: int = 0):
    """The same template plus its phase markers [(name, position)] and the kind
    of every allocation (param, data, act, grad, state, temp) -- what a CPU
    profile's annotations and the Analyzer's attribution provide (PAPER.md:212,
    240-246)."""
    T = _build(name, opt, zero_grad, streams, iterations, img, seq, micro)
    return T.arrays(), tuple(T.marks), tuple(T.kinds)


def _build(name, opt, zero_grad, streams, iterations, img, seq, micro):
    ops = model_ops(name, img, seq)
    T = _Tpl()
    s_data = 1 if streams else 0
    s_opt = 2 if streams else 0
    in_numel, in_es = input_numel(name, img, seq)
    params = []                 # (handle, shape)
    op_params = []
    for op in ops:
        hs = []
        for shp in op.params:
            h = T.alloc(shp[0] * shp[1] * F32, kind="param")
            params.append((h, shp))
            hs.append(len(params) - 1)
        op_params.append(hs)
    state = []
    if opt == "adagrad":        # Adagrad initialises its state in the constructor
        for (_, shp) in params:
            state += [T.alloc(x, kind="state") for x in _opt_state(opt, shp)]
    grads: Dict[int, int] = {}

    n = len(ops)
    sizes_in = []               # per-sample numel of each op's input
    cur = in_numel
    for op in ops:
        sizes_in.append(cur)
        if op.out:
            cur = op.out

    for it in range(iterations):
        T.mark("iter_start")
        if zero_grad == "pos1":
            T.mark("zg_start")
            for k in list(grads):
                T.free(grads.pop(k))
            T.mark("zg_end")
        T.mark("data_start")
        x = T.alloc(0, in_numel * in_es, s_data, kind="data")
        y = T.alloc(0, 8, s_data, kind="data")                    # labels
        T.mark("data_end")
        T.mark("fw_start")
        # ---- forward ----
        act = x                  # current activation handle
        act_owner = -1           # op index that produced act (-1 = batch data)
        saved: Dict[int, List[int]] = {}      # op index -> handles to free at its backward
        res_stack: List[Tuple[int, int]] = []
        for k, op in enumerate(ops):
            if op.res_start:
                res_stack.append((act, act_owner))
            ws = T.alloc(op.ws_fixed, op.ws) if (op.ws or op.ws_fixed) else None
            out = T.alloc(0, op.out * F32) if op.out else None
            ex = [T.alloc(f, p) for (f, p) in op.extra]
            T.free(ws)
            for _ in range(micro if op.out else 0):
                T.free(T.alloc(0, max(F32, op.out * F32 // 16)))
            saved.setdefault(k, []).extend(ex)
            if out is not None:
                in_saved = op.saves_in
                in_residual = any(h == act for h, _ in res_stack)
                if in_saved:
                    saved[k].append(act) if act != x else None
                elif not in_residual and act != x and not _kept(saved, act):
                    T.free(act)
                if op.res_add and res_stack:
                    h, owner = res_stack.pop()
                    if h != x and not _kept(saved, h) and h != act:
                        T.free(h)
                if op.saves_out:
                    saved[k].append(out)
                act, act_owner = out, k
        loss = T.alloc(F32)
        T.mark("fw_end")
        if zero_grad == "pos0":
            T.mark("zg_start")
            for k in list(grads):
                T.free(grads.pop(k))
            T.mark("zg_end")
        # ---- backward ----
        T.mark("bw_start")
        g = T.alloc(0, ops[-1].out * F32 if ops[-1].out else F32)
        if not _kept(saved, act) and act != x:
            T.free(act)
        for k in range(n - 1, -1, -1):
            op = ops[k]
            if op.out == 0:
                continue
            gi = T.alloc(0, sizes_in[k] * F32) if k > 0 else None
            if op.ws or op.ws_fixed:
                T.free(T.alloc(op.ws_fixed, op.ws))
            for _ in range(micro):
                T.free(T.alloc(0, max(F32, op.out * F32 // 16)))
            for pi in op_params[k]:
                h, shp = params[pi]
                if pi in grads:
                    T.free(T.alloc(shp[0] * shp[1] * F32))
                else:
                    grads[pi] = T.alloc(shp[0] * shp[1] * F32, kind="grad")
            for h in saved.pop(k, []):
                if h in T.live:
                    T.free(h)
            T.free(g)
            g = gi
        T.free(g)
        T.mark("bw_end")
        # ---- optimizer.step ----
        T.mark("opt_start")
        if it == 0 and opt != "adagrad":
            for (_, shp) in params:
                state += [T.alloc(x_, kind="state") for x_ in _opt_state(opt, shp)]
        for _ in range(_opt_temps(opt)):
            tmps = [T.alloc(shp[0] * shp[1] * F32, 0, s_opt, kind="temp") for (_, shp) in params]
            for h in tmps:
                T.free(h)
        T.mark("opt_end")
        for h in list(saved.values()):
            for hh in h:
                if hh in T.live:
                    T.free(hh)
        T.free(loss)
        T.free(y)
        T.free(x)
        T.mark("iter_end")
        # leftover activations (defensive)
    for k in list(grads):
        T.free(grads.pop(k))
    for h in state:
        T.free(h)
    for (h, _) in params:
        T.free(h)
    for h in list(T.live):
        T.free(h)
    return T


def _kept(saved: Dict[int, List[int]], h: int) -> bool:
    for v in saved.values():
        if h in v:
            return True
    return False


def instantiate(tpl, b: int, rng: Optional[np.random.Generator] = None, swap_p: float = 0.0):
    """bytes/tag arrays of one trace at batch size b, with optional seeded adjacent
    swaps (p per position) that emulate CPU-timing jitter (PAPER.md:248 footnote)."""
    sign, fixed, per, bid, stream = tpl
    nbytes = (fixed + per * int(b)) * sign
    tag = bid | (stream << np.uint32(28))
    if swap_p > 0 and rng is not None and len(nbytes) > 2:
        cand = np.flatnonzero(rng.random(len(nbytes) - 1) < swap_p)
        if len(cand):
            # non-overlapping: drop candidates adjacent to the previous one
            keep = np.ones(len(cand), bool)
            keep[1:] = np.diff(cand) > 1
            cand = cand[keep]
            same = bid[cand] == bid[cand + 1]
            cand = cand[~same]
            nbytes = nbytes.copy()
            tag = tag.copy()
            a, c = nbytes[cand].copy(), tag[cand].copy()
            nbytes[cand], tag[cand] = nbytes[cand + 1], tag[cand + 1]
            nbytes[cand + 1], tag[cand + 1] = a, c
    return nbytes.astype(np.int64), tag.astype(np.uint32)
