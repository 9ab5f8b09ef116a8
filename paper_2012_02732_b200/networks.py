"""Network definitions for the BASELINE configs.

* ``InceptionCell`` — the synthetic 3-branch Inception-style cell (8 ops on
  1x3x32x32; BASELINE.json configs[0]).
* ``NASNetAMobile`` — NASNet-A mobile (the Cadene
  reference implementation is not available offline).  Written from
  the published cell structure: stem conv → CellStem0/1 → 3 x (FirstCell +
  3 NormalCells) separated by 2 ReductionCells → ReLU → global pool → Linear,
  penultimate 1056 filters.  The CPU oracle runs this very module, so numeric
  parity does not depend on matching Cadene weight-for-weight.
* torchvision ResNet-50, Inception-v3 (aux_logits=False), MobileNetV2,
  EfficientNet-B0 through ``build_model``.

The "pad-then-slice" idioms of NASNet (factorized reduction path 2,
MaxPoolPad/AvgPoolPad, BranchSeparablesReduction) are small leaf modules with
an ``sw_spec()`` so the op-DAG builder lowers each to ONE kernel with shifted
padding instead of pad / op / slice copies; their CPU forward is the literal
pad → op → slice.
"""

from __future__ import annotations

import torch
import torch.nn as nn
import torch.nn.functional as F

BN_EPS = 1e-3


# --------------------------------------------------------------------------
# NASNet leaf modules with explicit lowering specs
# --------------------------------------------------------------------------

class PadPool(nn.Module):
    """ZeroPad2d((1,0,1,0)) → pool(3, s2, p1) → [:, :, 1:, 1:] (MaxPoolPad / AvgPoolPad)."""

    def __init__(self, mode: str):
        super().__init__()
        self.mode = mode

    def forward(self, x):
        x = F.pad(x, (1, 0, 1, 0))
        if self.mode == "max":
            x = F.max_pool2d(x, 3, stride=2, padding=1)
        else:
            x = F.avg_pool2d(x, 3, stride=2, padding=1, count_include_pad=False)
        return x[:, :, 1:, 1:]

    def sw_spec(self, in_shape):
        n, c, h, w = in_shape
        # padded input H+1 rows; pool out = floor((H+1+2-3)/2)+1; slice drops row 0.
        p = (h + 1 + 2 - 3) // 2 + 1 - 1
        q = (w + 1 + 2 - 3) // 2 + 1 - 1
        # kept window o' covers padded rows 2(o'+1)-1 .. +2 == input rows 2o' .. 2o'+2
        return {"kind": "pool", "mode": self.mode, "k": (3, 3), "stride": (2, 2), "pad": (0, 0),
                "out_hw": (p, q), "count_include_pad": False}


class SubsamplePath(nn.Module):
    """Factorized-reduction path: [shift] → AvgPool2d(1, s2) → 1x1 conv (no bias)."""

    def __init__(self, cin: int, cout: int, shift: bool):
        super().__init__()
        self.shift = shift
        self.conv = nn.Conv2d(cin, cout, 1, stride=1, bias=False)

    def forward(self, x):
        if self.shift:
            x = F.pad(x, (0, 1, 0, 1))[:, :, 1:, 1:]
        x = F.avg_pool2d(x, 1, stride=2, count_include_pad=False)
        return self.conv(x)

    def sw_spec(self, in_shape):
        n, c, h, w = in_shape
        p = (h - 1) // 2 + 1
        q = (w - 1) // 2 + 1
        off = -1 if self.shift else 0  # read x[2p+1, 2q+1] (zero past the edge)
        return {"kind": "conv", "module": self.conv, "stride": (2, 2), "pad": (off, off),
                "out_hw": (p, q)}


class PaddedDepthwise(nn.Module):
    """ZeroPad2d((1,0,1,0)) → depthwise conv(k, s, p) → [:, :, 1:, 1:]."""

    def __init__(self, ch: int, k: int, stride: int, pad: int):
        super().__init__()
        self.conv = nn.Conv2d(ch, ch, k, stride=stride, padding=pad, groups=ch, bias=False)

    def forward(self, x):
        x = F.pad(x, (1, 0, 1, 0))
        return self.conv(x)[:, :, 1:, 1:]

    def sw_spec(self, in_shape):
        n, c, h, w = in_shape
        k = self.conv.kernel_size[0]
        s = self.conv.stride[0]
        p = self.conv.padding[0]
        oh = (h + 1 + 2 * p - k) // s + 1 - 1
        ow = (w + 1 + 2 * p - k) // s + 1 - 1
        # output o' reads input rows o'*s + (s - p - 1) + r  → top pad p + 1 - s
        return {"kind": "dwconv", "module": self.conv, "stride": (s, s),
                "pad": (p + 1 - s, p + 1 - s), "out_hw": (oh, ow)}


# --------------------------------------------------------------------------
# NASNet-A building blocks
# --------------------------------------------------------------------------

def _bn(c):
    return nn.BatchNorm2d(c, eps=BN_EPS, momentum=0.1, affine=True)


class SepConv(nn.Module):
    def __init__(self, cin, cout, k, stride, pad, padded=False):
        super().__init__()
        if padded:
            self.depthwise = PaddedDepthwise(cin, k, stride, pad)
        else:
            self.depthwise = nn.Conv2d(cin, cin, k, stride=stride, padding=pad, groups=cin,
                                       bias=False)
        self.pointwise = nn.Conv2d(cin, cout, 1, bias=False)

    def forward(self, x):
        return self.pointwise(self.depthwise(x))


class BranchSep(nn.Module):
    """relu → sep(k, s) → bn → relu → sep(k, 1) → bn.  ``stem`` widens in the first sep."""

    def __init__(self, cin, cout, k, stride, pad, stem=False, padded=False):
        super().__init__()
        mid = cout if stem else cin
        self.relu = nn.ReLU()
        self.sep1 = SepConv(cin, mid, k, stride, pad, padded=padded)
        self.bn1 = _bn(mid)
        self.relu1 = nn.ReLU()
        self.sep2 = SepConv(mid, cout, k, 1, pad)
        self.bn2 = _bn(cout)

    def forward(self, x):
        x = self.bn1(self.sep1(self.relu(x)))
        return self.bn2(self.sep2(self.relu1(x)))


class ReluConvBn(nn.Sequential):
    def __init__(self, cin, cout):
        super().__init__(nn.ReLU(), nn.Conv2d(cin, cout, 1, bias=False), _bn(cout))


class FactorizedReduction(nn.Module):
    """relu → two shifted stride-2 1x1 paths → concat → bn (x_prev adjustment)."""

    def __init__(self, cin, cout):
        super().__init__()
        self.relu = nn.ReLU()
        self.path1 = SubsamplePath(cin, cout // 2, shift=False)
        self.path2 = SubsamplePath(cin, cout - cout // 2, shift=True)
        self.bn = _bn(cout)

    def forward(self, x):
        x = self.relu(x)
        return self.bn(torch.cat([self.path1(x), self.path2(x)], 1))


def _avg3():
    return nn.AvgPool2d(3, stride=1, padding=1, count_include_pad=False)


class CellStem0(nn.Module):
    def __init__(self, stem, f):
        super().__init__()
        self.conv_1x1 = ReluConvBn(stem, f)
        self.c0l = BranchSep(f, f, 5, 2, 2)
        self.c0r = BranchSep(stem, f, 7, 2, 3, stem=True)
        self.c1l = nn.MaxPool2d(3, stride=2, padding=1)
        self.c1r = BranchSep(stem, f, 7, 2, 3, stem=True)
        self.c2l = nn.AvgPool2d(3, stride=2, padding=1, count_include_pad=False)
        self.c2r = BranchSep(stem, f, 5, 2, 2, stem=True)
        self.c3r = _avg3()
        self.c4l = BranchSep(f, f, 3, 1, 1)
        self.c4r = nn.MaxPool2d(3, stride=2, padding=1)

    def forward(self, x):
        x1 = self.conv_1x1(x)
        i0 = self.c0l(x1) + self.c0r(x)
        i1 = self.c1l(x1) + self.c1r(x)
        i2 = self.c2l(x1) + self.c2r(x)
        i3 = self.c3r(i0) + i1
        i4 = self.c4l(i0) + self.c4r(x1)
        return torch.cat([i1, i2, i3, i4], 1)


class CellStem1(nn.Module):
    def __init__(self, stem, f):
        super().__init__()
        self.conv_1x1 = ReluConvBn(4 * (f // 2), f)
        self.reduce = FactorizedReduction(stem, f)
        self.c0l = BranchSep(f, f, 5, 2, 2)
        self.c0r = BranchSep(f, f, 7, 2, 3)
        self.c1l = nn.MaxPool2d(3, stride=2, padding=1)
        self.c1r = BranchSep(f, f, 7, 2, 3)
        self.c2l = nn.AvgPool2d(3, stride=2, padding=1, count_include_pad=False)
        self.c2r = BranchSep(f, f, 5, 2, 2)
        self.c3r = _avg3()
        self.c4l = BranchSep(f, f, 3, 1, 1)
        self.c4r = nn.MaxPool2d(3, stride=2, padding=1)

    def forward(self, x_conv0, x_stem0):
        left = self.conv_1x1(x_stem0)
        right = self.reduce(x_conv0)
        i0 = self.c0l(left) + self.c0r(right)
        i1 = self.c1l(left) + self.c1r(right)
        i2 = self.c2l(left) + self.c2r(right)
        i3 = self.c3r(i0) + i1
        i4 = self.c4l(i0) + self.c4r(left)
        return torch.cat([i1, i2, i3, i4], 1)


class NormalCell(nn.Module):
    """FirstCell when ``first`` (x_prev at twice the resolution → factorized reduction)."""

    def __init__(self, in_left, out_left, in_right, out_right, first=False):
        super().__init__()
        self.first = first
        if first:
            self.prev = FactorizedReduction(in_left, 2 * out_left)
            left_ch = 2 * out_left
        else:
            self.prev = ReluConvBn(in_left, out_left)
            left_ch = out_left
        self.conv_1x1 = ReluConvBn(in_right, out_right)
        self.c0l = BranchSep(out_right, out_right, 5, 1, 2)
        self.c0r = BranchSep(left_ch, left_ch, 3, 1, 1)
        self.c1l = BranchSep(left_ch, left_ch, 5, 1, 2)
        self.c1r = BranchSep(left_ch, left_ch, 3, 1, 1)
        self.c2l = _avg3()
        self.c3l = _avg3()
        self.c3r = _avg3()
        self.c4l = BranchSep(out_right, out_right, 3, 1, 1)

    def forward(self, x, x_prev):
        left = self.prev(x_prev)
        right = self.conv_1x1(x)
        i0 = self.c0l(right) + self.c0r(left)
        i1 = self.c1l(left) + self.c1r(left)
        i2 = self.c2l(right) + left
        i3 = self.c3l(left) + self.c3r(left)
        i4 = self.c4l(right) + right
        return torch.cat([left, i0, i1, i2, i3, i4], 1)


class ReductionCell(nn.Module):
    """``padded`` = ReductionCell0 (pad-then-slice ops), else ReductionCell1."""

    def __init__(self, in_left, out_left, in_right, out_right, padded):
        super().__init__()
        self.prev = ReluConvBn(in_left, out_left)
        self.conv_1x1 = ReluConvBn(in_right, out_right)
        c = out_right
        self.c0l = BranchSep(c, c, 5, 2, 2, padded=padded)
        self.c0r = BranchSep(c, c, 7, 2, 3, padded=padded)
        self.c1l = PadPool("max") if padded else nn.MaxPool2d(3, stride=2, padding=1)
        self.c1r = BranchSep(c, c, 7, 2, 3, padded=padded)
        self.c2l = PadPool("avg") if padded else nn.AvgPool2d(3, stride=2, padding=1,
                                                              count_include_pad=False)
        self.c2r = BranchSep(c, c, 5, 2, 2, padded=padded)
        self.c3r = _avg3()
        self.c4l = BranchSep(c, c, 3, 1, 1, padded=padded)
        self.c4r = PadPool("max") if padded else nn.MaxPool2d(3, stride=2, padding=1)

    def forward(self, x, x_prev):
        left = self.prev(x_prev)
        right = self.conv_1x1(x)
        i0 = self.c0l(right) + self.c0r(left)
        i1 = self.c1l(right) + self.c1r(left)
        i2 = self.c2l(right) + self.c2r(left)
        i3 = self.c3r(i0) + i1
        i4 = self.c4l(i0) + self.c4r(right)
        return torch.cat([i1, i2, i3, i4], 1)


class NASNetAMobile(nn.Module):
    """NASNet-A (4 @ 1056) mobile: 224x224 input, ~5.3 M params, ~0.6 B MACs."""

    def __init__(self, num_classes=1000, stem_filters=32, penultimate=1056, mult=2):
        super().__init__()
        f = penultimate // 24  # 44
        self.conv0 = nn.Sequential(nn.Conv2d(3, stem_filters, 3, stride=2, padding=0, bias=False),
                                   _bn(stem_filters))
        self.cell_stem_0 = CellStem0(stem_filters, f // (mult ** 2))
        self.cell_stem_1 = CellStem1(stem_filters, f // mult)
        self.cell_0 = NormalCell(f, f // 2, 2 * f, f, first=True)
        self.cell_1 = NormalCell(2 * f, f, 6 * f, f)
        self.cell_2 = NormalCell(6 * f, f, 6 * f, f)
        self.cell_3 = NormalCell(6 * f, f, 6 * f, f)
        self.reduction_cell_0 = ReductionCell(6 * f, 2 * f, 6 * f, 2 * f, padded=True)
        self.cell_6 = NormalCell(6 * f, f, 8 * f, 2 * f, first=True)
        self.cell_7 = NormalCell(8 * f, 2 * f, 12 * f, 2 * f)
        self.cell_8 = NormalCell(12 * f, 2 * f, 12 * f, 2 * f)
        self.cell_9 = NormalCell(12 * f, 2 * f, 12 * f, 2 * f)
        self.reduction_cell_1 = ReductionCell(12 * f, 4 * f, 12 * f, 4 * f, padded=False)
        self.cell_12 = NormalCell(12 * f, 2 * f, 16 * f, 4 * f, first=True)
        self.cell_13 = NormalCell(16 * f, 4 * f, 24 * f, 4 * f)
        self.cell_14 = NormalCell(24 * f, 4 * f, 24 * f, 4 * f)
        self.cell_15 = NormalCell(24 * f, 4 * f, 24 * f, 4 * f)
        self.relu = nn.ReLU()
        self.avg_pool = nn.AdaptiveAvgPool2d(1)
        self.dropout = nn.Dropout(0.5)
        self.last_linear = nn.Linear(24 * f, num_classes)

    def forward(self, x):
        c0 = self.conv0(x)
        s0 = self.cell_stem_0(c0)
        s1 = self.cell_stem_1(c0, s0)
        x0 = self.cell_0(s1, s0)
        x1 = self.cell_1(x0, s1)
        x2 = self.cell_2(x1, x0)
        x3 = self.cell_3(x2, x1)
        r0 = self.reduction_cell_0(x3, x2)
        x6 = self.cell_6(r0, x3)
        x7 = self.cell_7(x6, r0)
        x8 = self.cell_8(x7, x6)
        x9 = self.cell_9(x8, x7)
        r1 = self.reduction_cell_1(x9, x8)
        x12 = self.cell_12(r1, x9)
        x13 = self.cell_13(x12, r1)
        x14 = self.cell_14(x13, x12)
        x15 = self.cell_15(x14, x13)
        y = self.avg_pool(self.relu(x15))
        y = self.dropout(torch.flatten(y, 1))
        return self.last_linear(y)


class InceptionCell(nn.Module):
    """Synthetic 3-branch cell: stem 3x3 → {1x1 | 1x1→3x3 | maxpool→1x1} → concat → relu."""

    def __init__(self, cin=3, width=16, branch=16):
        super().__init__()
        self.stem = nn.Conv2d(cin, width, 3, padding=1)
        self.b1 = nn.Conv2d(width, branch, 1)
        self.b2a = nn.Conv2d(width, branch, 1)
        self.b2b = nn.Conv2d(branch, branch, 3, padding=1)
        self.pool = nn.MaxPool2d(3, stride=1, padding=1)
        self.b3 = nn.Conv2d(width, branch, 1)
        self.relu = nn.ReLU()

    def forward(self, x):
        s = self.stem(x)
        y = torch.cat([self.b1(s), self.b2b(self.b2a(s)), self.b3(self.pool(s))], 1)
        return self.relu(y)


# --------------------------------------------------------------------------
# factory
# --------------------------------------------------------------------------

CONFIGS = {
    # name: (input shape for batch 1, constructor)
    "cell": ((1, 3, 32, 32), lambda: InceptionCell()),
    "resnet50": ((1, 3, 224, 224), None),
    "inception_v3": ((1, 3, 299, 299), None),
    "nasnet_mobile": ((1, 3, 224, 224), lambda: NASNetAMobile()),
    "mobilenet_v2": ((1, 3, 32, 32), None),
    "efficientnet_b0": ((1, 3, 32, 32), None),
}


def randomize_bn(model: nn.Module, seed: int = 0) -> nn.Module:
    """Seeded non-trivial BN statistics so folding is exercised."""
    g = torch.Generator().manual_seed(seed + 12345)
    for m in model.modules():
        if isinstance(m, nn.BatchNorm2d):
            c = m.num_features
            with torch.no_grad():
                m.weight.copy_(torch.rand(c, generator=g) + 0.5)
                m.bias.copy_(torch.rand(c, generator=g) * 0.2 - 0.1)
                m.running_mean.copy_(torch.rand(c, generator=g) * 0.2 - 0.1)
                m.running_var.copy_(torch.rand(c, generator=g) + 0.5)
    return model


def calibrate_bn(model: nn.Module, shape, seed: int = 0, batch: int | None = None) -> nn.Module:
    """Set every BN's running statistics from one train-mode pass over a seeded
    N(0,1) calibration batch (cumulative average, i.e. exactly that batch's
    statistics), after ``randomize_bn`` drew the affine γ/β.

    Default random init makes deep nets explode in eval mode (torchvision
    Inception-v3's truncated-normal convs reach logits ~1e13, ResNet-50 ~1e3),
    which would turn the north_star's absolute gate into a relative one.  With
    calibrated statistics every BN output is ≈ γ·N(0,1) + β, so activations and
    logits stay O(1) and the unscaled rel 1e-3 / abs 1e-4 gate means what it
    says.  The statistics stay non-trivial (per-channel means and variances of
    a real forward), so BN folding is still exercised.  Small (CIFAR-sized)
    inputs reach 1x1 spatial extent in the last stages, so they calibrate on a
    larger batch: a per-channel variance taken over a handful of samples would
    amplify any other input."""
    if batch is None:
        batch = 4 if shape[-1] * shape[-2] >= 128 * 128 else 128
    g = torch.Generator().manual_seed(seed + 777)
    x = torch.randn((batch,) + tuple(shape[1:]), generator=g)
    bns = [m for m in model.modules() if isinstance(m, nn.BatchNorm2d)]
    saved = [m.momentum for m in bns]
    for m in bns:
        m.reset_running_stats()
        m.momentum = None
    model.train()
    with torch.no_grad():
        model(x)
    for m, mom in zip(bns, saved):
        m.momentum = mom
    return model.eval()


def build_model(name: str, seed: int = 0) -> tuple[nn.Module, tuple[int, ...]]:
    """Random-init model (eval mode, randomized BN affine, BN statistics
    calibrated on a seeded batch) and its batch-1 input shape."""
    torch.manual_seed(seed)
    shape, ctor = CONFIGS[name]
    if ctor is not None:
        model = ctor()
    else:
        import torchvision.models as tvm
        if name == "resnet50":
            model = tvm.resnet50(weights=None)
        elif name == "inception_v3":
            # PyTorch default init (as every other torchvision net here): with
            # init_weights=True (truncated normal, std 0.1) the fp32 CPU forward
            # itself misses the rel 1e-3 / abs 1e-4 gate against fp64 (ill-conditioned
            # head), so the gate would measure conditioning, not kernels
            model = tvm.inception_v3(weights=None, aux_logits=False, init_weights=False)
        elif name == "mobilenet_v2":
            model = tvm.mobilenet_v2(weights=None, num_classes=10)
        elif name == "efficientnet_b0":
            model = tvm.efficientnet_b0(weights=None, num_classes=10)
        else:
            raise KeyError(name)
    randomize_bn(model, seed)
    calibrate_bn(model, shape, seed)
    return model.eval(), shape


def example_input(shape, batch: int = 1, seed: int = 1) -> torch.Tensor:
    g = torch.Generator().manual_seed(seed)
    return torch.randn((batch,) + tuple(shape[1:]), generator=g)


TRAIN_CONFIGS = ("mobilenet_v2", "efficientnet_b0")


def build_train_model(name: str, seed: int = 0) -> nn.Module:
    """CIFAR-10-shaped training model (BASELINE config 5): torchvision
    MobileNetV2 / EfficientNet-B0 with 10 classes, random init, randomized BN
    affine, train mode.  Dropout and stochastic depth are set to p = 0: their
    RNG streams are not reproduced by the engine, and p = 0 keeps the step a
    deterministic function of (weights, batch) for the parity gate."""
    import torchvision.models as tvm
    torch.manual_seed(seed)
    if name == "mobilenet_v2":
        model = tvm.mobilenet_v2(weights=None, num_classes=10, dropout=0.0)
    elif name == "efficientnet_b0":
        model = tvm.efficientnet_b0(weights=None, num_classes=10, dropout=0.0, stochastic_depth_prob=0.0)
    else:
        raise KeyError(name)
    randomize_bn(model, seed)
    return model.train()


def train_batch(batch: int = 32, rank: int = 0, hw: int = 32):
    """Synthetic CIFAR-10 batch: randn images, labels seeded 1000+rank."""
    g = torch.Generator().manual_seed(1 + rank)
    x = torch.randn((batch, 3, hw, hw), generator=g)
    gl = torch.Generator().manual_seed(1000 + rank)
    y = torch.randint(0, 10, (batch,), generator=gl)
    return x, y
