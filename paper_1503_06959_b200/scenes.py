"""Seeded synthetic video for the BASELINE.json configs (stand-in datasets).

The paper measured on Stanford MAR / Rome Landmark sequences, which are not in
this container (reference SPEC.md:16).  BASELINE.json's five configs describe
seeded synthetic scenes instead; this module generates them with torch so the
same code runs on the CPU (parity fixtures, small configs) and on the GPU
(bench-scale batches, 64 x 1080p streams).  A (config, stream, device) triple
always yields the same bytes; CPU and CUDA RNG streams differ, so a parity
test generates on the CPU and uploads, and the bench's CPU baseline copies its
sample back from the GPU.

Scene model (BASELINE.json configs):
  * background: uniform noise, Gaussian-smoothed (sigma 1.5), rescaled to
    0..255, plus an optional coarse block layer (contrast at the 8-px scale
    the top-octave intensity mask sees);
  * objects: rectangles 60-120 px, checkerboard (cell 6-16 px, levels ~55/200)
    plus N(0, 20) texture noise, moving at a per-object speed in a random
    direction, bouncing off the frame edge, pasted at rounded positions;
  * optional global pan (bilinear resample of a larger canvas, then rounded);
  * per-frame additive Gaussian noise, rint, clip to uint8;
  * "fresh" kind (config 4): a new seeded texture every frame with 8x8 block
    offsets that change by >= 40 levels per frame, so every top-octave cell is
    selected.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class SceneConfig:
    width: int
    height: int
    n_frames: int
    n_streams: int = 1
    kind: str = "objects"  # objects | pan | static | fresh | mixed (s mod 3)
    n_objects: tuple[int, int] = (5, 5)  # inclusive range per stream
    speed: tuple[float, float] = (1.0, 3.0)  # px / frame
    pan_speed: tuple[float, float] = (0.5, 2.0)
    noise_sigma: float = 2.0
    block_contrast: float = 0.0  # amplitude of the coarse background block layer
    block_size: int = 24
    seed: int = 0


# BASELINE.json "configs" (index 0..4 -> config 1..5)
CONFIGS = {
    1: SceneConfig(640, 480, 100, 1, "objects", (5, 5), (1.0, 3.0), noise_sigma=2.0, seed=1),
    2: SceneConfig(1280, 720, 300, 1, "pan", (10, 10), (1.0, 3.0), (0.5, 2.0), noise_sigma=3.0,
                   block_contrast=120.0, block_size=24, seed=2),
    3: SceneConfig(1920, 1080, 200, 8, "objects", (5, 20), (0.0, 4.0), noise_sigma=2.0, seed=300),
    4: SceneConfig(3840, 2160, 120, 1, "fresh", (0, 0), (0.0, 0.0), noise_sigma=2.0, seed=400),
    5: SceneConfig(1920, 1080, 300, 64, "mixed", (5, 20), (0.0, 4.0), (0.5, 2.0), noise_sigma=2.0,
                   block_contrast=120.0, block_size=24, seed=500),
}


def _gauss_kernel(sigma: float, device) -> torch.Tensor:
    radius = int(4.0 * sigma + 0.5)  # scipy.ndimage default truncate=4.0
    x = torch.arange(-radius, radius + 1, dtype=torch.float32, device=device)
    k = torch.exp(-0.5 * (x / sigma) ** 2)
    return k / k.sum()


def _smooth(u: torch.Tensor, sigma: float) -> torch.Tensor:
    k = _gauss_kernel(sigma, u.device)
    r = (k.numel() - 1) // 2
    x = u[None, None]
    x = torch.nn.functional.pad(x, (r, r, 0, 0), mode="reflect")
    x = torch.nn.functional.conv2d(x, k.view(1, 1, 1, -1))
    x = torch.nn.functional.pad(x, (0, 0, r, r), mode="reflect")
    x = torch.nn.functional.conv2d(x, k.view(1, 1, -1, 1))
    return x[0, 0]


def _background(h: int, w: int, cfg: SceneConfig, g: torch.Generator, device) -> torch.Tensor:
    u = torch.rand((h, w), generator=g, device=device)
    s = _smooth(u, 1.5)
    b = 255.0 * (s - s.min()) / (s.max() - s.min())
    if cfg.block_contrast > 0:
        bs = cfg.block_size
        cells = torch.rand((h // bs + 1, w // bs + 1), generator=g, device=device) - 0.5
        blocks = cells.repeat_interleave(bs, 0).repeat_interleave(bs, 1)[:h, :w]
        b = 0.5 * b + 64.0 + 2.0 * cfg.block_contrast * blocks
    return b


def _object_texture(tw: int, th: int, g: torch.Generator, device) -> torch.Tensor:
    cell = int(torch.randint(6, 17, (1,), generator=g, device="cpu" if device is None else device).item())
    yy = torch.arange(th, device=device)[:, None] // cell
    xx = torch.arange(tw, device=device)[None, :] // cell
    lo = 55.0 + 20.0 * float(torch.rand((1,), generator=g, device=device).item())
    hi = 200.0 - 20.0 * float(torch.rand((1,), generator=g, device=device).item())
    chk = torch.where(((yy + xx) % 2) == 0, torch.full((), lo, device=device), torch.full((), hi, device=device))
    return (chk + 20.0 * torch.randn((th, tw), generator=g, device=device)).clamp(0, 255)


class SceneStream:
    """Deterministic frame source for one stream of a config."""

    def __init__(self, cfg: SceneConfig, stream: int, device="cpu"):
        self.cfg = cfg
        self.device = torch.device(device)
        self.stream = stream
        seed = cfg.seed + stream
        self.g = torch.Generator(device=self.device)
        self.g.manual_seed(seed)
        kind = cfg.kind
        if kind == "mixed":
            kind = ("static", "pan", "objects")[stream % 3]
        self.kind = kind
        W, H = cfg.width, cfg.height
        # geometry is drawn on a CPU generator so it does not depend on the device
        gc = torch.Generator().manual_seed(seed * 7919 + 17)
        self.gc = gc
        pad = 0
        if kind == "pan":
            smin, smax = cfg.pan_speed
            sp = smin + (smax - smin) * torch.rand((1,), generator=gc).item()
            ang = 2 * math.pi * torch.rand((1,), generator=gc).item()
            self.pan = (sp * math.cos(ang), sp * math.sin(ang))
            pad = int(math.ceil(max(smax, 1.0) * cfg.n_frames)) + 2
        else:
            self.pan = (0.0, 0.0)
        self.pad = pad
        if kind != "fresh":
            self.canvas = _background(H + 2 * pad, W + 2 * pad, cfg, self.g, self.device)
        lo, hi = cfg.n_objects
        n_obj = 0 if kind in ("fresh",) else int(torch.randint(lo, hi + 1, (1,), generator=gc).item())
        self.objects = []
        for _ in range(n_obj):
            tw = int(torch.randint(60, 121, (1,), generator=gc).item())
            th = int(torch.randint(60, 121, (1,), generator=gc).item())
            x0 = torch.rand((1,), generator=gc).item() * max(W - tw, 1)
            y0 = torch.rand((1,), generator=gc).item() * max(H - th, 1)
            if kind == "static":
                sp = 0.0
            else:
                sp = cfg.speed[0] + (cfg.speed[1] - cfg.speed[0]) * torch.rand((1,), generator=gc).item()
            ang = 2 * math.pi * torch.rand((1,), generator=gc).item()
            tex = _object_texture(tw, th, self.g, self.device)
            self.objects.append([x0, y0, sp * math.cos(ang), sp * math.sin(ang), tex])
        self.n = 0
        self._block_levels = None

    def _fresh_frame(self) -> torch.Tensor:
        cfg = self.cfg
        H, W = cfg.height, cfg.width
        u = torch.rand((H, W), generator=self.g, device=self.device)
        s = _smooth(u, 1.5)
        tex = 80.0 * (s - s.mean()) / (s.max() - s.min())
        bh, bw = -(-H // 8), -(-W // 8)
        if self._block_levels is None:
            lv = torch.randint(40, 216, (bh, bw), generator=self.g, device=self.device)
        else:
            step = torch.randint(45, 91, (bh, bw), generator=self.g, device=self.device)
            sign = torch.randint(0, 2, (bh, bw), generator=self.g, device=self.device) * 2 - 1
            lv = self._block_levels + sign * step
            lv = torch.where((lv < 40) | (lv > 215), self._block_levels - sign * step, lv)
        self._block_levels = lv
        blocks = lv.float().repeat_interleave(8, 0).repeat_interleave(8, 1)[:H, :W]
        return blocks + tex

    def next_frame(self) -> torch.Tensor:
        """The next uint8 (H, W) frame on this stream's device."""
        cfg = self.cfg
        H, W = cfg.height, cfg.width
        n = self.n
        if self.kind == "fresh":
            img = self._fresh_frame()
        elif self.kind == "pan":
            ox = self.pad + self.pan[0] * n
            oy = self.pad + self.pan[1] * n
            ix, iy = int(math.floor(ox)), int(math.floor(oy))
            fx, fy = ox - ix, oy - iy
            c = self.canvas
            a = c[iy:iy + H, ix:ix + W]
            b = c[iy:iy + H, ix + 1:ix + 1 + W]
            d = c[iy + 1:iy + 1 + H, ix:ix + W]
            e = c[iy + 1:iy + 1 + H, ix + 1:ix + 1 + W]
            img = (1 - fy) * ((1 - fx) * a + fx * b) + fy * ((1 - fx) * d + fx * e)
            img = torch.floor(img + 0.5)
        else:
            img = self.canvas.clone()
        for ob in self.objects:
            x0, y0, vx, vy, tex = ob
            th, tw = tex.shape
            xi, yi = int(round(x0)), int(round(y0))
            xa, ya = max(xi, 0), max(yi, 0)
            xb, yb = min(xi + tw, W), min(yi + th, H)
            if xa < xb and ya < yb:
                img[ya:yb, xa:xb] = tex[ya - yi:yb - yi, xa - xi:xb - xi]
            # advance with bounce
            x0 += vx
            y0 += vy
            if x0 < 0 or x0 > W - tw:
                vx = -vx
                x0 = min(max(x0, 0.0), float(max(W - tw, 0)))
            if y0 < 0 or y0 > H - th:
                vy = -vy
                y0 = min(max(y0, 0.0), float(max(H - th, 0)))
            ob[0], ob[1], ob[2], ob[3] = x0, y0, vx, vy
        if cfg.noise_sigma > 0:
            img = img + cfg.noise_sigma * torch.randn((H, W), generator=self.g, device=self.device)
        self.n += 1
        return torch.round(img).clamp(0, 255).to(torch.uint8)


def generate(cfg: SceneConfig, n_frames: int | None = None, streams=None, device="cpu") -> torch.Tensor:
    """uint8 tensor [S, N, H, W] of the first n_frames of the given streams."""
    n_frames = cfg.n_frames if n_frames is None else n_frames
    streams = range(cfg.n_streams) if streams is None else streams
    out = []
    for s in streams:
        st = SceneStream(cfg, s, device)
        out.append(torch.stack([st.next_frame() for _ in range(n_frames)]))
    return torch.stack(out)
