"""Synthetic allocation traces: the reference's generators plus the
layer-shape CNN traces and random sweeps the B200 benchmarks use.

* ``GenSpec`` / ``cnn_like_trace`` / ``rnn_like_trace`` / ``rnn_epoch_lengths``
  / ``generate`` reproduce the reference generators (workloads.py:24-133)
  draw for draw — tests pin their output text by SHA-256 against traces the
  reference produced (tests/golden/traces.json).
* ``uniform_blocks`` / ``walk_trace``: the random-lifetime and alloc/free
  random-walk families of SURVEY.md §8(d) item 5.
* ``net_trace``: training-iteration traces built from layer shapes (AlexNet,
  GoogLeNet, ResNet-50, Inception-ResNet-v2; BASELINE.json configs 1-3):
  forward keeps every layer output, convolutions take an 8 MB workspace
  (PAPER.md:593-597), backward allocates input/weight gradients layer by
  layer in reverse and releases activations as soon as they are consumed.
"""

from __future__ import annotations

import random
from dataclasses import dataclass


@dataclass(frozen=True)
class GenSpec:
    model: str  # "cnn" | "rnn"
    layers: int = 8
    batch: int = 32
    seed: int = 0
    variable_length: tuple | None = None
    workspace: bool = True
    untimed: bool = False

    def __post_init__(self) -> None:
        if self.model not in ("cnn", "rnn"):
            raise ValueError(f"model must be 'cnn' or 'rnn', got {self.model!r}")
        if self.layers < 1:
            raise ValueError(f"layers must be >= 1, got {self.layers}")
        if self.batch < 1:
            raise ValueError(f"batch must be >= 1, got {self.batch}")
        if self.variable_length is not None:
            lo, hi = self.variable_length
            if not 1 <= lo <= hi:
                raise ValueError(f"bad length range {self.variable_length}")


class _TraceWriter:
    """Accumulates trace lines and hands out allocation references."""

    def __init__(self, header: str):
        self.lines = [header]
        self.nref = 0

    def a(self, size: int, label: str | None = None) -> int:
        self.lines.append(f"A {size} {label}" if label else f"A {size}")
        self.nref += 1
        return self.nref

    def f(self, ref: int) -> None:
        self.lines.append(f"F {ref}")

    def raw(self, line: str) -> None:
        self.lines.append(line)

    def text(self) -> str:
        return "\n".join(self.lines) + "\n"


def _scaled(batch: int, base: float, draw: float) -> int:
    return batch * max(8, round(base * draw))


def cnn_like_trace(spec: GenSpec) -> str:
    """Nested forward/backward activations (layer i freed at backward step
    2L-i), shrinking with depth, plus a growing one-tick workspace per layer."""
    rng = random.Random(spec.seed)
    w = _TraceWriter(f"# cnn-like: layers={spec.layers} batch={spec.batch} seed={spec.seed}")
    acts = []
    for i in range(1, spec.layers + 1):
        acts.append(w.a(_scaled(spec.batch, 2048 * 0.88 ** min(i, 64),
                                rng.uniform(0.75, 1.3)), f"act{i}"))
        if spec.workspace:
            grow = 1.0 + 4.0 * i / (i + 12.0)
            w.f(w.a(_scaled(spec.batch, 320 * grow, rng.uniform(0.85, 1.2)), f"ws{i}"))
    for ref in reversed(acts):
        w.f(ref)
    return w.text()


def rnn_epoch_lengths(spec: GenSpec, epochs: int) -> list:
    lo, hi = spec.variable_length if spec.variable_length else (16, 16)
    rng = random.Random(f"{spec.seed}-lengths")
    return [rng.randint(lo, hi) for _ in range(epochs)]


def rnn_like_trace(spec: GenSpec, length: int) -> str:
    """Fixed event structure; only the sequence buffer scales with length."""
    if length < 1:
        raise ValueError(f"length must be >= 1, got {length}")
    rng = random.Random(spec.seed)
    states = [_scaled(spec.batch, 512, rng.uniform(0.7, 1.4)) for _ in range(spec.layers)]
    temps = [_scaled(spec.batch, 96, rng.uniform(0.5, 1.6)) for _ in range(spec.layers)]
    beam = _scaled(spec.batch, 640, rng.uniform(0.8, 1.2))
    w = _TraceWriter(f"# rnn-like: layers={spec.layers} batch={spec.batch} "
                     f"seed={spec.seed} length={length}")
    seq = w.a(spec.batch * 64 * length, "seq")
    held = []
    for i in range(1, spec.layers + 1):
        held.append(w.a(states[i - 1], f"h{i}"))
        w.f(w.a(temps[i - 1], f"tmp{i}"))
    if spec.untimed:
        w.raw("I")
        w.f(w.a(beam, "beam"))
        w.raw("R")
    for ref in reversed(held):
        w.f(ref)
    w.f(seq)
    return w.text()


def generate(spec: GenSpec) -> str:
    if spec.model == "cnn":
        return cnn_like_trace(spec)
    return rnn_like_trace(spec, rnn_epoch_lengths(spec, 1)[0])


# ---------------------------------------------------------------------------
# random sweeps
# ---------------------------------------------------------------------------
def uniform_blocks(n: int, seed: int = 0, max_size: int = 1 << 20) -> list:
    """(size, alloc, free) with alloc ~ U{0..2n-1}, free ~ U{alloc+1..2n}."""
    r = random.Random(seed)
    out = []
    for _ in range(n):
        a = r.randint(0, 2 * n - 1)
        f = r.randint(a + 1, 2 * n)
        out.append((r.randint(1, max_size), a, f))
    return out


def uniform_arrays(n: int, seed: int = 0, max_size: int = 1 << 20):
    """numpy-generated uniform family for large sweeps (not the oracle draw)."""
    import numpy as np
    g = np.random.default_rng(seed)
    a = g.integers(0, 2 * n, n, dtype=np.int64)
    f = a + 1 + (g.integers(0, 1 << 62, n, dtype=np.int64) % (2 * n - a))
    s = g.integers(1, max_size + 1, n, dtype=np.int64)
    return a, f, s


def walk_trace(n: int, seed: int = 0, p_free: float = 0.45, max_size: int = 1 << 20) -> str:
    """Alloc/free random walk: n allocations; each step frees a random live
    block with probability p_free (when any is live)."""
    r = random.Random(seed)
    w = _TraceWriter("")
    w.lines.clear()
    live = []
    while w.nref < n:
        if live and r.random() < p_free:
            w.f(live.pop(r.randrange(len(live))))
        else:
            live.append(w.a(r.randint(1, max_size)))
    return w.text()


# ---------------------------------------------------------------------------
# layer-shape training traces (BASELINE.json configs 1-3)
# ---------------------------------------------------------------------------
WORKSPACE_BYTES = 8 * 1024 * 1024
F32 = 4


@dataclass
class _Layer:
    name: str
    out: tuple            # (C, H, W)
    inputs: list          # indices of producer layers (-1 = network input)
    params: int = 0       # weight + bias elements
    conv: bool = False


class _Net:
    def __init__(self, name: str, c: int, h: int, w: int):
        self.name = name
        self.input = (c, h, w)
        self.layers: list = []

    def _add(self, name, out, inputs, params=0, conv=False) -> int:
        self.layers.append(_Layer(name, out, list(inputs), params, conv))
        return len(self.layers) - 1

    def shape(self, i: int) -> tuple:
        return self.input if i < 0 else self.layers[i].out

    def conv(self, src, cout, k, stride=1, pad=None, name="conv", kw=None, bn=False, relu=True):
        c, h, w = self.shape(src)
        kh, kwid = k, (kw if kw is not None else k)
        ph = (kh - 1) // 2 if pad is None else pad
        pw = (kwid - 1) // 2 if pad is None else pad
        ho = (h + 2 * ph - kh) // stride + 1
        wo = (w + 2 * pw - kwid) // stride + 1
        x = self._add(name, (cout, ho, wo), [src], c * cout * kh * kwid + cout, conv=True)
        if bn:
            x = self._add(name + "/bn", (cout, ho, wo), [x], 2 * cout)
        if relu:
            x = self._add(name + "/relu", (cout, ho, wo), [x])
        return x

    def pool(self, src, k, stride, pad=0, name="pool", global_=False):
        c, h, w = self.shape(src)
        if global_:
            return self._add(name, (c, 1, 1), [src])
        ho = (h + 2 * pad - k) // stride + 1
        wo = (w + 2 * pad - k) // stride + 1
        return self._add(name, (c, ho, wo), [src])

    def lrn(self, src, name="lrn"):
        return self._add(name, self.shape(src), [src])

    def fc(self, src, cout, name="fc", relu=False):
        c, h, w = self.shape(src)
        x = self._add(name, (cout, 1, 1), [src], c * h * w * cout + cout)
        if relu:
            x = self._add(name + "/relu", (cout, 1, 1), [x])
        return x

    def concat(self, srcs, name="concat"):
        c = sum(self.shape(s)[0] for s in srcs)
        _, h, w = self.shape(srcs[0])
        return self._add(name, (c, h, w), srcs)

    def add(self, a, b, name="add", relu=True):
        x = self._add(name, self.shape(a), [a, b])
        if relu:
            x = self._add(name + "/relu", self.shape(a), [x])
        return x


def _alexnet() -> _Net:
    n = _Net("alexnet", 3, 227, 227)
    x = n.conv(-1, 96, 11, 4, 0, "conv1")
    x = n.pool(n.lrn(x, "norm1"), 3, 2, name="pool1")
    x = n.conv(x, 256, 5, 1, 2, "conv2")
    x = n.pool(n.lrn(x, "norm2"), 3, 2, name="pool2")
    x = n.conv(x, 384, 3, name="conv3")
    x = n.conv(x, 384, 3, name="conv4")
    x = n.conv(x, 256, 3, name="conv5")
    x = n.pool(x, 3, 2, name="pool5")
    x = n.fc(x, 4096, "fc6", relu=True)
    x = n.fc(x, 4096, "fc7", relu=True)
    n.fc(x, 1000, "fc8")
    return n


def _googlenet() -> _Net:
    n = _Net("googlenet", 3, 224, 224)
    x = n.conv(-1, 64, 7, 2, 3, "conv1")
    x = n.lrn(n.pool(x, 3, 2, 0, "pool1"), "norm1")
    x = n.conv(x, 64, 1, name="conv2r")
    x = n.conv(x, 192, 3, name="conv2")
    x = n.pool(n.lrn(x, "norm2"), 3, 2, 0, "pool2")
    table = [("3a", 64, 96, 128, 16, 32, 32), ("3b", 128, 128, 192, 32, 96, 64), "pool",
             ("4a", 192, 96, 208, 16, 48, 64), ("4b", 160, 112, 224, 24, 64, 64),
             ("4c", 128, 128, 256, 24, 64, 64), ("4d", 112, 144, 288, 32, 64, 64),
             ("4e", 256, 160, 320, 32, 128, 128), "pool",
             ("5a", 256, 160, 320, 32, 128, 128), ("5b", 384, 192, 384, 48, 128, 128)]
    for row in table:
        if row == "pool":
            x = n.pool(x, 3, 2, 0, "pool")
            continue
        tag, c1, c3r, c3, c5r, c5, cp = row
        b1 = n.conv(x, c1, 1, name=f"i{tag}/1x1")
        b2 = n.conv(n.conv(x, c3r, 1, name=f"i{tag}/3x3r"), c3, 3, name=f"i{tag}/3x3")
        b3 = n.conv(n.conv(x, c5r, 1, name=f"i{tag}/5x5r"), c5, 5, name=f"i{tag}/5x5")
        b4 = n.conv(n.pool(x, 3, 1, 1, f"i{tag}/pool"), cp, 1, name=f"i{tag}/proj")
        x = n.concat([b1, b2, b3, b4], f"i{tag}/out")
    x = n.pool(x, 7, 1, name="pool5", global_=True)
    n.fc(x, 1000, "loss3")
    return n


def _resnet50() -> _Net:
    n = _Net("resnet50", 3, 224, 224)
    x = n.conv(-1, 64, 7, 2, 3, "conv1", bn=True)
    x = n.pool(x, 3, 2, 1, "pool1")
    for stage, (blocks, width) in enumerate([(3, 64), (4, 128), (6, 256), (3, 512)]):
        for b in range(blocks):
            stride = 2 if (b == 0 and stage > 0) else 1
            tag = f"res{stage + 2}{chr(97 + b)}"
            y = n.conv(x, width, 1, stride, 0, f"{tag}/a", bn=True)
            y = n.conv(y, width, 3, 1, 1, f"{tag}/b", bn=True)
            y = n.conv(y, 4 * width, 1, 1, 0, f"{tag}/c", bn=True, relu=False)
            sc = n.conv(x, 4 * width, 1, stride, 0, f"{tag}/proj", bn=True, relu=False) \
                if b == 0 else x
            x = n.add(y, sc, f"{tag}/add")
    x = n.pool(x, 7, 1, name="pool5", global_=True)
    n.fc(x, 1000, "fc1000")
    return n


def _inception_resnet_v2() -> _Net:
    n = _Net("inception_resnet_v2", 3, 299, 299)

    def c(src, cout, k, stride=1, pad=None, name="c", kw=None):
        return n.conv(src, cout, k, stride, pad, name, kw=kw, bn=True)

    x = c(-1, 32, 3, 2, 0, "stem1")
    x = c(x, 32, 3, 1, 0, "stem2")
    x = c(x, 64, 3, 1, 1, "stem3")
    x = n.pool(x, 3, 2, 0, "stem_pool1")
    x = c(x, 80, 1, 1, 0, "stem4")
    x = c(x, 192, 3, 1, 0, "stem5")
    x = n.pool(x, 3, 2, 0, "stem_pool2")
    b0 = c(x, 96, 1, name="m5b/b0")
    b1 = c(c(x, 48, 1, name="m5b/b1a"), 64, 5, name="m5b/b1b")
    b2 = c(c(c(x, 64, 1, name="m5b/b2a"), 96, 3, name="m5b/b2b"), 96, 3, name="m5b/b2c")
    b3 = c(n.pool(x, 3, 1, 1, "m5b/pool"), 64, 1, name="m5b/b3")
    x = n.concat([b0, b1, b2, b3], "m5b")
    for i in range(10):  # Inception-ResNet-A, 35x35x320
        t = f"a{i}"
        b0 = c(x, 32, 1, name=f"{t}/b0")
        b1 = c(c(x, 32, 1, name=f"{t}/b1a"), 32, 3, name=f"{t}/b1b")
        b2 = c(c(c(x, 32, 1, name=f"{t}/b2a"), 48, 3, name=f"{t}/b2b"), 64, 3, name=f"{t}/b2c")
        up = n.conv(n.concat([b0, b1, b2], f"{t}/cat"), 320, 1, name=f"{t}/up", relu=False)
        x = n.add(x, up, f"{t}/add")
    b0 = c(x, 384, 3, 2, 0, "m6a/b0")
    b1 = c(c(c(x, 256, 1, name="m6a/b1a"), 256, 3, name="m6a/b1b"), 384, 3, 2, 0, "m6a/b1c")
    b2 = n.pool(x, 3, 2, 0, "m6a/pool")
    x = n.concat([b0, b1, b2], "m6a")
    for i in range(20):  # Inception-ResNet-B, 17x17x1088
        t = f"b{i}"
        b0 = c(x, 192, 1, name=f"{t}/b0")
        b1 = c(c(c(x, 128, 1, name=f"{t}/b1a"), 160, 1, name=f"{t}/b1b", kw=7),
               192, 7, name=f"{t}/b1c", kw=1)
        up = n.conv(n.concat([b0, b1], f"{t}/cat"), 1088, 1, name=f"{t}/up", relu=False)
        x = n.add(x, up, f"{t}/add")
    b0 = c(c(x, 256, 1, name="m7a/b0a"), 384, 3, 2, 0, "m7a/b0b")
    b1 = c(c(x, 256, 1, name="m7a/b1a"), 288, 3, 2, 0, "m7a/b1b")
    b2 = c(c(c(x, 256, 1, name="m7a/b2a"), 288, 3, name="m7a/b2b"), 320, 3, 2, 0, "m7a/b2c")
    b3 = n.pool(x, 3, 2, 0, "m7a/pool")
    x = n.concat([b0, b1, b2, b3], "m7a")
    for i in range(10):  # Inception-ResNet-C, 8x8x2080
        t = f"c{i}"
        b0 = c(x, 192, 1, name=f"{t}/b0")
        b1 = c(c(c(x, 192, 1, name=f"{t}/b1a"), 224, 1, name=f"{t}/b1b", kw=3),
               256, 3, name=f"{t}/b1c", kw=1)
        up = n.conv(n.concat([b0, b1], f"{t}/cat"), 2080, 1, name=f"{t}/up", relu=False)
        x = n.add(x, up, f"{t}/add", relu=(i < 9))
    x = c(x, 1536, 1, name="conv7b")
    x = n.pool(x, 8, 1, name="avgpool", global_=True)
    n.fc(x, 1000, "logits")
    return n


NETS = {"alexnet": _alexnet, "googlenet": _googlenet, "resnet50": _resnet50,
        "inception_resnet_v2": _inception_resnet_v2}


def net_trace(net: str, batch: int) -> str:
    """One training iteration of `net` at mini-batch `batch` as trace text.

    Forward: every layer output stays live until backward consumes it; each
    convolution borrows an 8 MB workspace for its own duration.  Backward (in
    reverse layer order): the output gradient of a layer is complete once all
    consumers ran; the layer allocates gradients for each input (accumulated
    into an existing buffer when an input fans out), a weight gradient that
    is applied and released immediately, a workspace for convolutions, then
    releases its output gradient and its output activation."""
    if net not in NETS:
        raise ValueError(f"unknown net {net!r}; choose from {sorted(NETS)}")
    if batch < 1:
        raise ValueError("batch must be >= 1")
    g = NETS[net]()
    w = _TraceWriter(f"# net: {g.name} batch={batch}")
    elems = lambda shp: shp[0] * shp[1] * shp[2]  # noqa: E731
    x_in = w.a(batch * elems(g.input) * F32, "input")
    out_ref = []
    for lay in g.layers:
        out_ref.append(w.a(batch * elems(lay.out) * F32, lay.name))
        if lay.conv:
            w.f(w.a(WORKSPACE_BYTES, lay.name + "/ws"))
    loss = w.a(F32 * batch, "loss")
    grad = {len(g.layers) - 1: w.a(batch * elems(g.layers[-1].out) * F32, "gy")}
    w.f(loss)
    grad_in = None
    for li in range(len(g.layers) - 1, -1, -1):
        lay = g.layers[li]
        for src in lay.inputs:
            if src < 0:
                if grad_in is None:
                    grad_in = w.a(batch * elems(g.input) * F32, "gx")
            elif src not in grad:
                grad[src] = w.a(batch * elems(g.shape(src)) * F32, f"g/{g.layers[src].name}")
        if lay.params:
            w.f(w.a(lay.params * F32, lay.name + "/gW"))
        if lay.conv:
            w.f(w.a(WORKSPACE_BYTES, lay.name + "/bws"))
        w.f(grad.pop(li))
        w.f(out_ref[li])
    if grad_in is not None:
        w.f(grad_in)
    w.f(x_in)
    return w.text()


def lstm_profiles(count: int, layers: int = 6, batch: int = 64, seed: int = 2024,
                  length_range: tuple = (10, 50)) -> list:
    """BASELINE.json config 4: `count` variable-length LSTM seq2seq profiles
    (rnn_like_trace over the seeded epoch lengths)."""
    spec = GenSpec(model="rnn", layers=layers, batch=batch, seed=seed,
                   variable_length=length_range)
    return [rnn_like_trace(spec, ell) for ell in rnn_epoch_lengths(spec, count)]
