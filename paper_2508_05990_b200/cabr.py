"""Context-aware block refinement (drop-in for ``bayermc.cabr``, cabr.py:1-399).

The network forward pass, patch extraction, the weight-free ring vote and the
block write-back run on the GPU (``csrc/bmc_cabr.cu`` through the C ABI in
include/bmc_ext.h).  Weight bookkeeping -- the tensor spec, seeded/zero
initialisation and the flat weight-file format -- is host data handling and
keeps the reference's exact layout and messages, so weight files and seeded
weights are interchangeable with the reference's.

Numerics: the reference evaluates the convolutions as float32 einsums
(cabr.py:206-216); the kernel evaluates the same float32 products and sums in a
different association order, so logits agree to float32 rounding
(tests: ``|d| <= 1e-5 * max|logit| + 1e-6``), not bit for bit, and a label can
differ only where the reference's two best logits are that close.
"""

from __future__ import annotations

import json
import struct
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .frame_io import Frame, LabelMap

CONTEXT_MASK = 16
_ENC_WIDTHS = (16, 32, 32)
_ENC_STRIDES = (2, 2, 1)
_DEC_WIDTH = 32
_UPSAMPLE = 4
_MAGIC_NOTE = "little-endian float32 payload"


def _require_block_size(block_size: int) -> None:
    if block_size < CONTEXT_MASK:
        raise ValueError(
            f"CaBR block size must be at least {CONTEXT_MASK}: the fixed "
            f"{CONTEXT_MASK}x{CONTEXT_MASK} context mask would cover a "
            f"{block_size}x{block_size} block entirely")


def _require_kernel_block(block_size: int) -> None:
    _require_block_size(block_size)
    if block_size % 16:
        raise NotImplementedError(f"the B200 CaBR kernel takes block sizes that are multiples of 16, got {block_size}")


@dataclass(frozen=True, eq=False)
class CabrPatch:
    """Inputs for one flagged block: image window and masked one-hot context (cabr.py:43-57)."""

    image: np.ndarray    # (1, 2K+1, 2K+1) float32 in [0, 1]
    context: np.ndarray  # (num_classes, 2K+1, 2K+1) float32 one-hot
    block_size: int

    def __post_init__(self):
        side = 2 * self.block_size + 1
        if self.image.shape != (1, side, side):
            raise ValueError(f"image patch must be (1, {side}, {side})")
        if self.context.ndim != 3 or self.context.shape[1:] != (side, side):
            raise ValueError(f"context patch must be (C, {side}, {side})")


# ---------------------------------------------------------------------------
# Weights (cabr.py:97-199): host data handling, reference layout
# ---------------------------------------------------------------------------

def weight_spec(num_classes: int) -> list:
    """(name, shape) for every tensor, in canonical order."""
    spec = []
    cin = 1
    for i, cout in enumerate(_ENC_WIDTHS):
        spec += [(f"img_enc.{i}.weight", (cout, cin, 3, 3)), (f"img_enc.{i}.bias", (cout,))]
        cin = cout
    cin = num_classes
    for i, cout in enumerate(_ENC_WIDTHS):
        spec += [(f"ctx_enc.{i}.weight", (cout, cin, 3, 3)), (f"ctx_enc.{i}.bias", (cout,))]
        cin = cout
    spec += [("dec.0.weight", (_DEC_WIDTH, 2 * _ENC_WIDTHS[-1], 3, 3)), ("dec.0.bias", (_DEC_WIDTH,)),
             ("dec.1.weight", (_DEC_WIDTH, _DEC_WIDTH, 3, 3)), ("dec.1.bias", (_DEC_WIDTH,)),
             ("head.weight", (num_classes, _DEC_WIDTH, 1, 1)), ("head.bias", (num_classes,))]
    return spec


@dataclass(frozen=True, eq=False)
class CabrWeights:
    tensors: dict

    def __post_init__(self):
        expected = dict(weight_spec(self.num_classes))
        if set(self.tensors) != set(expected):
            missing = sorted(set(expected) - set(self.tensors))
            extra = sorted(set(self.tensors) - set(expected))
            raise ValueError(f"weight tensors mismatch: missing {missing}, extra {extra}")
        for name, shape in expected.items():
            t = self.tensors[name]
            if tuple(t.shape) != shape:
                raise ValueError(f"{name}: expected shape {shape}, got {tuple(t.shape)}")
            if t.dtype != np.float32:
                raise ValueError(f"{name}: weights must be float32")

    @property
    def num_classes(self) -> int:
        head = self.tensors.get("head.weight")
        if head is None:
            raise ValueError("missing decoder head tensor")
        return int(head.shape[0])

    def payload(self) -> np.ndarray:
        """Every tensor in weight_spec order, flattened and concatenated (the weight file's payload)."""
        return np.concatenate([np.ascontiguousarray(self.tensors[n], dtype="<f4").reshape(-1)
                               for n, _ in weight_spec(self.num_classes)])


def random_weights(num_classes: int, seed: int = 0, scale: float = 0.05) -> CabrWeights:
    rng = np.random.default_rng(seed)
    return CabrWeights(tensors={name: (rng.standard_normal(shape) * scale).astype(np.float32)
                                for name, shape in weight_spec(num_classes)})


def zero_weights(num_classes: int) -> CabrWeights:
    return CabrWeights(tensors={name: np.zeros(shape, dtype=np.float32) for name, shape in weight_spec(num_classes)})


def save_weights(weights: CabrWeights, path) -> None:
    """Write ``<header-length:u32><JSON header><raw float32 payload>`` (cabr.py:152-168)."""
    entries, payload = [], bytearray()
    for name, _ in weight_spec(weights.num_classes):
        tensor = weights.tensors[name]
        entries.append({"name": name, "shape": list(tensor.shape), "offset": len(payload)})
        payload.extend(tensor.astype("<f4").tobytes())
    header = json.dumps({"tensors": entries, "note": _MAGIC_NOTE}).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(struct.pack("<I", len(header)))
        fh.write(header)
        fh.write(bytes(payload))


def load_weights(path) -> CabrWeights:
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < 4:
        raise ValueError(f"{path}: truncated weight file")
    (header_len,) = struct.unpack_from("<I", raw, 0)
    if 4 + header_len > len(raw):
        raise ValueError(f"{path}: header length exceeds file size")
    header = json.loads(raw[4:4 + header_len].decode("utf-8"))
    payload = raw[4 + header_len:]
    tensors = {}
    for entry in header["tensors"]:
        shape = tuple(int(s) for s in entry["shape"])
        count = int(np.prod(shape)) if shape else 1
        offset = int(entry["offset"])
        if offset + 4 * count > len(payload):
            raise ValueError(f"{path}: tensor {entry['name']} overruns the payload")
        tensors[entry["name"]] = np.frombuffer(payload, dtype="<f4", count=count, offset=offset) \
            .reshape(shape).astype(np.float32)
    return CabrWeights(tensors=tensors)


# Device copies of weights, re-laid out for the kernel once per (weights, device).
_PACKED = weakref.WeakKeyDictionary()


def packed_weights(weights: CabrWeights, torch, dev):
    """The weights on ``dev`` in the kernel's layout (bmc_cabr_pack_weights); cached."""
    per = _PACKED.setdefault(weights, {})
    key = str(dev)
    if key not in per:
        C = weights.num_classes
        src = torch.from_numpy(weights.payload()).to(dev)
        need = sum(int(np.prod(shape)) for _, shape in weight_spec(C))
        if src.numel() != need:
            raise ValueError(f"weight payload holds {src.numel()} floats, the network needs {need}")
        # the packed layout adds the decoder's merged row taps (bmc_cabr_weight_floats)
        dst = torch.empty(N.load().bmc_cabr_weight_floats(C), dtype=torch.float32, device=dev)
        N.check(N.load().bmc_cabr_pack_weights(N.ptr(src), C, N.ptr(dst), N.stream_handle()))
        per[key] = dst
    return per[key]


# ---------------------------------------------------------------------------
# Device inputs
# ---------------------------------------------------------------------------

def _pixels_on_device(frame, torch, dev):
    """(tensor, pixel_kind) of a Frame (uint8 0 / uint16 1, divided on device by the
    dtype maximum, cabr.py:72-73) or a 2-D array already in [0, 1] (float32 2)."""
    if isinstance(frame, Frame):
        data = np.ascontiguousarray(frame.data)
        kind = 0 if data.dtype == np.uint8 else 1
        t = torch.from_numpy(np.array(data.view(np.int16) if kind == 1 else data, copy=True)).to(dev)
        return t, kind
    arr = np.ascontiguousarray(np.asarray(frame, dtype=np.float32))
    return torch.from_numpy(arr).to(dev), 2


def _frame_shape(frame):
    return (frame.height, frame.width) if isinstance(frame, Frame) else np.asarray(frame).shape


def _origins(blocks, torch, dev):
    arr = np.asarray([(int(x), int(y)) for x, y in blocks], dtype=np.int32).reshape(-1, 2)
    return arr, torch.from_numpy(arr).to(dev)


def extract_patch(frame, labels: LabelMap, block_origin, block_size: int) -> CabrPatch:
    """Build the image/context patch pair for the block at ``block_origin`` (cabr.py:60-90), on the GPU."""
    _require_block_size(block_size)
    if tuple(_frame_shape(frame)) != labels.classes.shape:
        raise ValueError("frame and label map dimensions differ")
    torch = N.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    pix, kind = _pixels_on_device(frame, torch, dev)
    lab = torch.from_numpy(np.ascontiguousarray(labels.classes)).to(dev)
    _, org = _origins([block_origin], torch, dev)
    side = 2 * block_size + 1
    C = labels.num_classes
    img = torch.empty((1, 1, side, side), dtype=torch.float32, device=dev)
    ctx = torch.empty((1, C, side, side), dtype=torch.float32, device=dev)
    N.check(N.load().bmc_cabr_extract_patches(N.ptr(pix), kind, N.ptr(lab), labels.height, labels.width, N.ptr(org),
                                              1, int(block_size), C, N.ptr(img), N.ptr(ctx), N.stream_handle()))
    return CabrPatch(image=img[0].cpu().numpy(), context=ctx[0].cpu().numpy(), block_size=block_size)


# ---------------------------------------------------------------------------
# Forward pass (cabr.py:206-250)
# ---------------------------------------------------------------------------

def cabr_forward(patch: CabrPatch, weights: CabrWeights) -> np.ndarray:
    """Class logits of shape (num_classes, K, K) for the patch's block (fp32, on the GPU)."""
    num_classes = weights.num_classes
    if patch.context.shape[0] != num_classes:
        raise ValueError(f"context patch has {patch.context.shape[0]} channels, weights expect {num_classes}")
    k = patch.block_size
    _require_kernel_block(k)
    torch = N.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    img = torch.from_numpy(np.ascontiguousarray(patch.image, dtype=np.float32)).to(dev)
    ctx = torch.from_numpy(np.ascontiguousarray(patch.context, dtype=np.float32)).to(dev)
    out = torch.empty((1, num_classes, k, k), dtype=torch.float32, device=dev)
    N.check(N.load().bmc_cabr_forward_patches(N.ptr(img), N.ptr(ctx), 1, k, num_classes,
                                              N.ptr(packed_weights(weights, torch, dev)), N.ptr(out), None,
                                              N.stream_handle()))
    return out[0].cpu().numpy()


def cabr_forward_blocks(frame, labels: LabelMap, blocks, block_size: int, weights: CabrWeights):
    """Batched ``cabr_forward(extract_patch(frame, labels, o, K), weights)`` over ``blocks``:
    returns (logits (n, C, K, K) float32, argmax labels (n, K, K) uint8)."""
    _require_kernel_block(block_size)
    if weights.num_classes != labels.num_classes:
        raise ValueError("weights and label map disagree on num_classes")
    if tuple(_frame_shape(frame)) != labels.classes.shape:
        raise ValueError("frame and label map dimensions differ")
    torch = N.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    pix, kind = _pixels_on_device(frame, torch, dev)
    lab = torch.from_numpy(np.ascontiguousarray(labels.classes)).to(dev)
    arr, org = _origins(blocks, torch, dev)
    n, C, k = len(arr), labels.num_classes, int(block_size)
    logits = torch.empty((n, C, k, k), dtype=torch.float32, device=dev)
    arg = torch.empty((n, k, k), dtype=torch.uint8, device=dev)
    N.check(N.load().bmc_cabr_forward_blocks(N.ptr(pix), kind, N.ptr(lab), labels.height, labels.width, N.ptr(org), n,
                                             k, C, N.ptr(packed_weights(weights, torch, dev)), N.ptr(logits),
                                             N.ptr(arg), N.stream_handle()))
    return logits.cpu().numpy(), arg.cpu().numpy()


# ---------------------------------------------------------------------------
# Block application (cabr.py:306-345)
# ---------------------------------------------------------------------------

def refine_blocks(frame, labels: LabelMap, blocks, block_size: int, weights: CabrWeights | None = None) -> LabelMap:
    """Re-label the flagged blocks; pixels outside them are untouched.

    ``blocks`` lists pixel-coordinate block origins (x, y).  With ``weights`` the
    network's argmax replaces each block; without, the ring-vote fallback does.
    Every block reads the input labels; write-back is clipped to the frame and
    in list order, as the reference's loop.
    """
    blocks = [(int(x), int(y)) for x, y in blocks]
    if not blocks:
        return labels
    _require_block_size(block_size)
    if any(x < 0 or y < 0 for x, y in blocks):
        raise ValueError("block origins must be non-negative")
    if weights is not None:
        if weights.num_classes != labels.num_classes:
            raise ValueError("weights and label map disagree on num_classes")
        _require_kernel_block(block_size)
        if tuple(_frame_shape(frame)) != labels.classes.shape:
            raise ValueError("frame and label map dimensions differ")
    torch = N.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    H, W = labels.height, labels.width
    lab = torch.from_numpy(np.ascontiguousarray(labels.classes)).to(dev)
    out = torch.empty_like(lab)
    arr, org = _origins(blocks, torch, dev)
    n, k = len(arr), int(block_size)
    staging = torch.empty(n * k * k, dtype=torch.uint8, device=dev)
    owner = torch.empty(H * W, dtype=torch.int32, device=dev)
    if weights is not None:
        pix, kind = _pixels_on_device(frame, torch, dev)
        packed, flagged = packed_weights(weights, torch, dev), None
    else:
        pix, kind, packed = None, 0, None
        flagged = torch.empty(H * W, dtype=torch.uint8, device=dev)
    N.check(N.load().bmc_refine_blocks(N.ptr(pix), kind, N.ptr(lab), N.ptr(out), H, W, N.ptr(org), n, k,
                                       labels.num_classes, N.ptr(packed), N.ptr(staging), N.ptr(owner),
                                       N.ptr(flagged), N.stream_handle()))
    return LabelMap(width=W, height=H, classes=out.cpu().numpy(), num_classes=labels.num_classes)


# ---------------------------------------------------------------------------
# FLOPs accounting (cabr.py:352-399)
# ---------------------------------------------------------------------------

def _conv_out(size: int, kernel: int, stride: int, pad: int) -> int:
    return (size + 2 * pad - kernel) // stride + 1


def layer_flops(block_size: int, num_classes: int) -> list:
    """(layer name, flops) per convolution for one forward invocation: 2*kh*kw*Cin*Cout*Hout*Wout."""
    _require_block_size(block_size)
    side = 2 * block_size + 1
    layers = []
    for prefix, cin in (("img_enc", 1), ("ctx_enc", num_classes)):
        size = side
        for i, (cout, stride) in enumerate(zip(_ENC_WIDTHS, _ENC_STRIDES)):
            size = _conv_out(size, 3, stride, 1)
            layers.append((f"{prefix}.{i}", 2 * 3 * 3 * cin * cout * size * size))
            cin = cout
    size = _conv_out(size, 3, 1, 1)
    layers.append(("dec.0", 2 * 3 * 3 * 2 * _ENC_WIDTHS[-1] * _DEC_WIDTH * size * size))
    size = _conv_out(size * _UPSAMPLE, 3, 1, 1)
    layers.append(("dec.1", 2 * 3 * 3 * _DEC_WIDTH * _DEC_WIDTH * size * size))
    layers.append(("head", 2 * _DEC_WIDTH * num_classes * size * size))
    return layers


def _regions(k: int, t0: int, ts: int):
    """Receptive field of block output rows [t0, t0+ts) per layer (csrc/bmc_cabr.cu regions())."""
    nd = k // 2 + 1
    l0 = k // 2 + 2 + t0
    d0 = ((l0 - 1) >> 2, ((l0 + ts) >> 2) + 1)
    e2 = (max(d0[0] - 1, 0), min(d0[1] + 1, nd))
    e1 = (max(e2[0] - 1, 0), min(e2[1] + 1, nd))
    e0 = (max(2 * e1[0] - 1, 0), min(2 * (e1[1] - 1) + 2, k + 1))
    return {"e0": e0[1] - e0[0], "e1": e1[1] - e1[0], "e2": e2[1] - e2[0], "d0": d0[1] - d0[0]}


def executed_flops(block_size: int, num_classes: int) -> int:
    """FLOPs the B200 kernel executes per block (2 per multiply-add): every layer only
    over the receptive field of the cropped K x K logits, per 32 x 32 output tile
    (the reference's layer_flops counts the full maps)."""
    _require_kernel_block(block_size)
    k, c = block_size, num_classes
    ts = 32 if k >= 32 else 16
    total = 0
    for ty in range(0, k, ts):
        ry = _regions(k, ty, ts)
        for tx in range(0, k, ts):
            rx = _regions(k, tx, ts)
            a = {n: ry[n] * rx[n] for n in ry}
            total += 2 * 9 * 16 * a["e0"]                     # img_enc.0 (ctx_enc.0 is a table lookup)
            total += 2 * (2 * 9 * 16 * 32 * a["e1"])          # img/ctx enc.1
            total += 2 * (2 * 9 * 32 * 32 * a["e2"])          # img/ctx enc.2
            total += 2 * 9 * 64 * 32 * a["d0"]                # dec.0
            # dec.1: rows u % 4 in {1, 2} read one dec.0 row (3 merged taps), the others 9 taps
            total += 2 * 6 * 32 * 32 * ts * ts + 2 * 32 * c * ts * ts  # dec.1 + head
    return total


def count_cabr_flops(block_size: int, num_classes: int, invocations: int) -> int:
    """Total flops for ``invocations`` forward passes."""
    if invocations < 0:
        raise ValueError("invocation count must be >= 0")
    return sum(f for _, f in layer_flops(block_size, num_classes)) * invocations
