"""Seeded synthetic Bayer clips for tests and the benchmark.

The reference ships only luma generators (synth.py:18-104); the Bayer clip
recipe here follows SURVEY.md §8d: three seeded value-noise channels on a
canvas larger than the frame, cropped at (m + vx*t, m + vy*t) per frame and
point-sampled through the CFA (frame_io.mosaic_rgb).  Even velocities keep the
CFA phase (plane MV = v/2); odd velocities break it (the stress case).
``value_noise`` restates the reference's generator (synth.py:18-41) so clips
built here equal clips built from the reference's own noise.
"""

from __future__ import annotations

import numpy as np

from .frame_io import Frame, FrameKind, LabelMap, mosaic_rgb


def value_noise(width: int, height: int, seed: int, cell: int = 16, detail: float = 0.15) -> np.ndarray:
    """Bilinear random lattice + per-pixel detail, scaled to uint8."""
    rng = np.random.default_rng(seed)
    lattice = rng.random((height // cell + 2, width // cell + 2))
    fy_all = np.arange(height) / cell
    fx_all = np.arange(width) / cell
    iy = fy_all.astype(np.int64)
    ix = fx_all.astype(np.int64)
    fy = (fy_all - iy)[:, None]
    fx = (fx_all - ix)[None, :]
    y0, x0 = iy[:, None], ix[None, :]
    # same left-to-right association as synth.py:36 so values match bit for bit
    smooth = (lattice[y0, x0] * (1 - fy) * (1 - fx) + lattice[y0, x0 + 1] * (1 - fy) * fx
              + lattice[y0 + 1, x0] * fy * (1 - fx) + lattice[y0 + 1, x0 + 1] * fy * fx)
    noise = smooth * (1 - detail) + rng.random((height, width)) * detail
    return np.clip(noise * 255.0, 0, 255).astype(np.uint8)


def bayer_pan_clip(width: int, height: int, frames: int, velocity, seed: int = 0,
                   pattern: FrameKind = FrameKind.BAYER_RGGB, dtype=np.uint8, square: int = 0,
                   square_velocity=(0, 0)) -> np.ndarray:
    """(frames, height, width) raw Bayer clip of a textured pan.

    ``square`` > 0 pastes a separately textured square moving with
    ``square_velocity`` (pixels/frame, relative to the frame) on top.
    """
    vx, vy = int(velocity[0]), int(velocity[1])
    m = max(abs(vx), abs(vy)) * frames + 8
    wc, hc = width + 2 * m, height + 2 * m
    chans = [value_noise(wc, hc, seed + k) for k in range(3)]
    if square:
        patch = [(value_noise(square, square, seed + 10 + k, cell=8) // 2 + 112).astype(np.uint8) for k in range(3)]
        sx0, sy0 = width // 4, height // 4
    out = np.empty((frames, height, width), dtype=np.uint16 if np.dtype(dtype) == np.uint16 else np.uint8)
    for t in range(frames):
        x, y = m + vx * t, m + vy * t
        rgb = [c[y:y + height, x:x + width].copy() for c in chans]
        if square:
            qx = sx0 + square_velocity[0] * t
            qy = sy0 + square_velocity[1] * t
            qx = min(max(qx, 0), width - square)
            qy = min(max(qy, 0), height - square)
            for c, p in zip(rgb, patch):
                c[qy:qy + square, qx:qx + square] = p
        data = mosaic_rgb(*rgb, pattern=pattern).data
        out[t] = data.astype(np.uint16) * 257 if out.dtype == np.uint16 else data
    return out


# full-res velocity sweep (px/frame); odd steps are added on alternate segments
C5_SWEEP = (0, 2, 8, 16, 24, 40, 64, 96, 200)


def bayer_path_clip(width: int, height: int, path, seed: int = 0, pattern: FrameKind = FrameKind.BAYER_RGGB,
                    dtype=np.uint8, square: int = 0, square_velocity=(0, 0)) -> np.ndarray:
    """Like ``bayer_pan_clip`` but the crop origin follows ``path`` (one (x, y) full-res
    offset per frame, any integers), so the pan velocity can change from frame to frame."""
    path = [(int(x), int(y)) for x, y in path]
    xs, ys = [p[0] for p in path], [p[1] for p in path]
    mx, my = -min(xs) + 8, -min(ys) + 8
    wc, hc = width + mx + max(xs) + 8, height + my + max(ys) + 8
    chans = [value_noise(wc, hc, seed + k) for k in range(3)]
    if square:
        patch = [(value_noise(square, square, seed + 10 + k, cell=8) // 2 + 112).astype(np.uint8) for k in range(3)]
        sx0, sy0 = width // 4, height // 4
    out = np.empty((len(path), height, width), dtype=np.uint16 if np.dtype(dtype) == np.uint16 else np.uint8)
    for t, (px, py) in enumerate(path):
        x, y = mx + px, my + py
        rgb = [c[y:y + height, x:x + width].copy() for c in chans]
        if square:
            qx = min(max(sx0 + square_velocity[0] * t, 0), width - square)
            qy = min(max(sy0 + square_velocity[1] * t, 0), height - square)
            for c, p in zip(rgb, patch):
                c[qy:qy + square, qx:qx + square] = p
        data = mosaic_rgb(*rgb, pattern=pattern).data
        out[t] = data.astype(np.uint16) * 257 if out.dtype == np.uint16 else data
    return out


def c5_clip(width: int = 1920, height: int = 1080, frames: int = 40, seed: int = 7, cut_at: int = 30,
            dtype=np.uint8) -> np.ndarray:
    """high-motion Bayer sweep with a moving textured square and a scene cut.

    Frames before ``cut_at`` pan with a piecewise-constant velocity stepping through
    ``C5_SWEEP`` (three frames per step; odd steps +1 on alternate segments, vertical
    component -vx/3), with a 192-px square moving at (13, -7); from ``cut_at`` on an
    unrelated scene pans at (24, -16)."""
    path, x, y = [], 0, 0
    for t in range(cut_at):
        if t:
            k = min((t - 1) // 3, len(C5_SWEEP) - 1)
            vx = C5_SWEEP[k] + (k % 2)
            x, y = x + vx, y - vx // 3
        path.append((x, y))
    a = bayer_path_clip(width, height, path, seed=seed, dtype=dtype, square=192, square_velocity=(13, -7))
    if frames <= cut_at:
        return a[:frames]
    b = bayer_pan_clip(width, height, frames - cut_at, (24, -16), seed=seed + 1000, dtype=dtype)
    return np.concatenate([a, b])


def scene_cut_clip(width: int, height: int, frames: int, cut_at: int, seed: int = 0, dtype=np.uint8) -> np.ndarray:
    """Static textured Bayer scene A before ``cut_at``, unrelated scene B after."""
    a = bayer_pan_clip(width, height, 1, (0, 0), seed, dtype=dtype)[0]
    b = bayer_pan_clip(width, height, 1, (0, 0), seed + 1000003, dtype=dtype)[0]
    return np.stack([a if t < cut_at else b for t in range(frames)])


def gen_translating_scene(width: int, height: int, frames: int, velocity, seed: int = 0, square_size: int = 48,
                          start=None, fg_class: int = 1):
    """Textured luma square over a textured background with exact labels
    (restates synth.py:44-85 so the SPEC acceptance sequences are identical)."""
    vx, vy = int(velocity[0]), int(velocity[1])
    if frames < 1:
        raise ValueError("need at least one frame")
    if square_size >= min(width, height):
        raise ValueError("square must fit inside the frame")
    sx0, sy0 = (width // 4, height // 4) if start is None else (int(start[0]), int(start[1]))
    for t in (0, frames - 1):
        x, y = sx0 + vx * t, sy0 + vy * t
        if x < 0 or y < 0 or x + square_size > width or y + square_size > height:
            raise ValueError(f"square leaves the frame at t={t}: origin ({x}, {y})")
    background = value_noise(width, height, seed)
    patch = (value_noise(square_size, square_size, seed + 1, cell=8) // 2 + 112).astype(np.uint8)
    out_frames, out_labels = [], []
    for t in range(frames):
        x, y = sx0 + vx * t, sy0 + vy * t
        pixels = background.copy()
        pixels[y:y + square_size, x:x + square_size] = patch
        classes = np.zeros((height, width), dtype=np.uint8)
        classes[y:y + square_size, x:x + square_size] = fg_class
        out_frames.append(Frame(width=width, height=height, data=pixels, kind=FrameKind.LUMA))
        out_labels.append(LabelMap(width=width, height=height, classes=classes, num_classes=max(2, fg_class + 1)))
    return out_frames, out_labels


def gen_scene_cut(width: int, height: int, frames: int, cut_at: int, seed: int = 0) -> list:
    """Two unrelated static luma scenes joined at ``cut_at`` (restates synth.py:88-104)."""
    if frames < 1:
        raise ValueError("need at least one frame")
    scene_a = value_noise(width, height, seed)
    scene_b = value_noise(width, height, seed + 1000003)
    return [Frame(width=width, height=height, data=(scene_a if t < cut_at else scene_b).copy(), kind=FrameKind.LUMA)
            for t in range(frames)]


def frames_of(clip: np.ndarray, pattern: FrameKind = FrameKind.BAYER_RGGB) -> list:
    return [Frame(width=c.shape[1], height=c.shape[0], data=c, kind=pattern) for c in clip]


def block_labels(width: int, height: int, frames: int, num_classes: int = 19, seed: int = 0) -> list:
    """Per-frame synthetic key-frame label maps (stand-ins for backbone output)."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, num_classes, (height // 8 + 1, width // 8 + 1)).astype(np.uint8)
    out = []
    for t in range(frames):
        cls = np.kron(np.roll(base, t, axis=1), np.ones((8, 8), np.uint8))[:height, :width]
        out.append(LabelMap(width=width, height=height, classes=np.ascontiguousarray(cls), num_classes=num_classes))
    return out
