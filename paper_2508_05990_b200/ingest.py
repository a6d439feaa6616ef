"""Bayer file ingest onto the GPU.

The reference reads frames one at a time on the host (frame_io.py:202-291:
binary PGM parsed with numpy, 16-bit payloads byte-swapped by
``np.frombuffer(dtype=">u2").astype(uint16)``; PNG through Pillow).  Here the
file payloads of a whole clip land in ONE pinned host buffer exactly as they
are stored, cross PCIe once, and are decoded by ``bmc_unpack_raw`` straight
into the (T, H, W) uint16 clip buffer the motion engine reads:

* 16-bit PGM (big-endian): 2 bytes/px on the wire, byte swap on the GPU;
* 8-bit PGM: the payload IS the frame (no decode);
* 10/12-bit MIPI CSI-2 packed raw (RAW10: 4 px in 5 bytes, RAW12: 2 px in
  3 bytes) -- 1.25 / 1.5 bytes per pixel on the wire instead of 2.

``frame_io.load_frame`` uses the same decode for 16-bit PGMs, so the drop-in
returns the reference's Frame bit for bit.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from . import _native as N

FORMATS = {"be16": N.RAW_BE16, "raw10": N.RAW_MIPI10, "raw12": N.RAW_MIPI12}


def parse_pgm_header(raw: bytes, path) -> tuple:
    """(width, height, maxval, payload offset) of a binary PGM (frame_io.py:202-229),
    with the reference's error messages."""
    if raw[:2] != b"P5":
        raise ValueError(f"{path}: not a binary PGM (P5) file")
    pos, tokens = 2, []
    while len(tokens) < 3:
        while pos < len(raw) and raw[pos:pos + 1].isspace():
            pos += 1
        if pos < len(raw) and raw[pos:pos + 1] == b"#":
            while pos < len(raw) and raw[pos:pos + 1] != b"\n":
                pos += 1
            continue
        start = pos
        while pos < len(raw) and not raw[pos:pos + 1].isspace():
            pos += 1
        if start == pos:
            raise ValueError(f"{path}: truncated PGM header")
        tokens.append(raw[start:pos])
    width, height, maxval = (int(t) for t in tokens)
    if maxval <= 0 or maxval > 65535:
        raise ValueError(f"{path}: unsupported PGM maxval {maxval}")
    return width, height, maxval, pos + 1  # a single whitespace byte follows maxval


def packed_row_bytes(width: int, fmt: str) -> int:
    if fmt == "be16":
        return 2 * width
    if fmt == "raw10":
        return (width + 3) // 4 * 5
    if fmt == "raw12":
        return (width + 1) // 2 * 3
    raise ValueError(f"unknown packed format {fmt!r}; expected one of {sorted(FORMATS)}")


def decode(payload, width: int, height: int, fmt: str, *, frames: int = 1, row_bytes: int | None = None,
           frame_bytes: int | None = None, shift: int = 0, out=None):
    """Decode ``frames`` packed payloads (host bytes / ndarray / tensor; pinned host
    memory gives an asynchronous copy) into a (frames, height, width) uint16 device
    tensor (``out`` if given) with ``bmc_unpack_raw``."""
    torch = N.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    rb = packed_row_bytes(width, fmt) if row_bytes is None else int(row_bytes)
    fb = rb * height if frame_bytes is None else int(frame_bytes)
    if isinstance(payload, torch.Tensor):
        src = payload.reshape(-1)
    else:
        host = (np.frombuffer(payload, dtype=np.uint8) if isinstance(payload, (bytes, bytearray, memoryview))
                else np.ascontiguousarray(payload).reshape(-1).view(np.uint8))
        src = torch.from_numpy(host if host.flags.writeable else host.copy())
    if src.numel() < fb * (frames - 1) + rb * height:
        raise ValueError(f"payload of {src.numel()} bytes is shorter than {frames} frame(s) of {width}x{height} {fmt}")
    src_dev = src.to(dev, non_blocking=bool(src.is_pinned())) if src.device.type != "cuda" else src
    if out is None:
        out = torch.empty((frames, height, width), dtype=torch.uint16, device=dev)
    N.check(N.load().bmc_unpack_raw(N.ptr(src_dev), fb, rb, int(frames), int(height), int(width), FORMATS[fmt],
                                    int(shift), N.ptr(out), N.stream_handle()))
    return out


def encode_be16(frames_u16):
    """uint16 frames -> big-endian payload bytes (the PGM 16-bit body, frame_io.py:238-242)
    on the GPU; returns a host uint8 ndarray."""
    torch = N.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    src = frames_u16 if isinstance(frames_u16, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(frames_u16, dtype=np.uint16))
    src = src.to(dev).contiguous()
    out = torch.empty(src.numel() * 2, dtype=torch.uint8, device=dev)
    N.check(N.load().bmc_pack_be16(N.ptr(src), src.numel(), N.ptr(out), N.stream_handle()))
    return out.cpu().numpy()


def pack_mipi(frames: np.ndarray, bits: int) -> np.ndarray:
    """Host encoder of MIPI RAW10/RAW12 payloads (test/fixture helper: cameras
    produce these; the product decodes them).  frames: (..., H, W) codes < 2**bits."""
    a = np.asarray(frames, dtype=np.uint16)
    if bits == 10:
        if a.shape[-1] % 4:
            raise ValueError("RAW10 packing needs a width divisible by 4")
        g = a.reshape(*a.shape[:-1], -1, 4)
        msb = (g >> 2).astype(np.uint8)
        lsb = ((g[..., 0] & 3) | ((g[..., 1] & 3) << 2) | ((g[..., 2] & 3) << 4) | ((g[..., 3] & 3) << 6))
        return np.concatenate([msb, lsb[..., None].astype(np.uint8)], axis=-1).reshape(*a.shape[:-1], -1)
    if bits == 12:
        if a.shape[-1] % 2:
            raise ValueError("RAW12 packing needs an even width")
        g = a.reshape(*a.shape[:-1], -1, 2)
        msb = (g >> 4).astype(np.uint8)
        lsb = ((g[..., 0] & 15) | ((g[..., 1] & 15) << 4)).astype(np.uint8)
        return np.concatenate([msb, lsb[..., None]], axis=-1).reshape(*a.shape[:-1], -1)
    raise ValueError("bits must be 10 or 12")


class PgmClipReader:
    """Read a list of binary PGM files of one size into a reusable pinned buffer
    (payloads as stored) and decode them on the GPU into a (T, H, W) device clip
    (uint8 for maxval < 256, uint16 otherwise) -- the streaming ingest for
    ``ClipEngine.load_frames`` / ``ClipSession.run``."""

    def __init__(self):
        self._pin = None
        self._done = None  # event after the last copy out of the pinned buffer

    def read(self, paths):
        torch = N.require_cuda()
        if self._done is not None:
            self._done.synchronize()  # the previous clip's H2D has left the pinned buffer
        paths = [Path(p) for p in paths]
        if not paths:
            raise ValueError("empty frame list")
        heads, blobs = [], []
        for p in paths:
            raw = p.read_bytes()
            w, h, mx, off = parse_pgm_header(raw, p)
            bpp = 1 if mx < 256 else 2
            if len(raw) - off < w * h * bpp:
                raise ValueError(f"{p}: PGM payload shorter than header promises")
            heads.append((w, h, bpp))
            blobs.append(memoryview(raw)[off:off + w * h * bpp])
        if len(set(heads)) != 1:
            raise ValueError("all frames of a clip must share size and bit depth")
        w, h, bpp = heads[0]
        need = len(paths) * w * h * bpp
        if self._pin is None or self._pin.numel() < need:
            self._pin = torch.empty(need, dtype=torch.uint8).pin_memory()
        host = self._pin[:need].numpy()
        for i, b in enumerate(blobs):
            host[i * w * h * bpp:(i + 1) * w * h * bpp] = np.frombuffer(b, dtype=np.uint8)
        dev = torch.device("cuda", torch.cuda.current_device())
        if bpp == 1:
            out = self._pin[:need].to(dev, non_blocking=True).reshape(len(paths), h, w)
        else:
            out = decode(self._pin[:need], w, h, "be16", frames=len(paths))
        self._done = torch.cuda.Event()
        self._done.record()
        return out
