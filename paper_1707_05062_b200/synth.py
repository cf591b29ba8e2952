"""Seeded synthetic inputs for the five BASELINE.json configs (C1-C5).

The paper's images (Lenna, Tulips, a YFCC100M clip) are not
available, so these generators stand in for them with the shapes and value
distributions BASELINE.json names.  Deterministic for a given (seed, device,
torch version); every config has a fixed default seed recorded in CONFIGS.
Generated with torch ops (device-agnostic); the GPU path and the CPU
reference always consume the very same bytes.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

LEVELS_C1 = (20, 55, 90, 125, 160, 195, 230)


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    w: int
    h: int
    seed: int
    desc: str

    @property
    def pixels(self) -> int:
        return self.n * self.w * self.h


CONFIGS = {
    "C1": Config("C1", 1, 512, 512, 0x51C1, "512x512 7-region Voronoi, levels {20..230}, N(0,8^2)"),
    "C2": Config("C2", 1, 5184, 3456, 0x51C2,
                 "5184x3456 gradient 0-200 + 40 ellipses (+-60) + N(0,5^2)"),
    "C3": Config("C3", 512, 1920, 1080, 0x51C3,
                 "512 frames 1920x1080, 12-region Voronoi drifting 2 px/frame + N(0,6^2)"),
    "C4": Config("C4", 1, 16384, 16384, 0x51C4, "16384x16384 i.i.d. uniform u8"),
    "C5": Config("C5", 65536, 128, 128, 0x51C5,
                 "65536 x 128x128: stripes {0,128,255} / constant / 0-255 checker / bimodal N(60|190,15^2)"),
}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _to_u8(x: torch.Tensor) -> torch.Tensor:
    return torch.round(x).clamp_(0, 255).to(torch.uint8)


def _voronoi_labels(w: int, h: int, sx: torch.Tensor, sy: torch.Tensor) -> torch.Tensor:
    dev = sx.device
    xs = torch.arange(w, device=dev, dtype=torch.float32)
    ys = torch.arange(h, device=dev, dtype=torch.float32)
    dx = (xs[None, :] - sx[:, None]) ** 2            # (k, w)
    dy = (ys[None, :] - sy[:, None]) ** 2            # (k, h)
    d = dy[:, :, None] + dx[:, None, :]              # (k, h, w)
    return torch.argmin(d, dim=0)


def c1(seed: int = CONFIGS["C1"].seed, device="cpu", w: int = 512, h: int = 512) -> torch.Tensor:
    """7 Voronoi regions, levels from LEVELS_C1, + N(0, 8^2)."""
    g = _gen(seed, device)
    sx = torch.rand(7, generator=g, device=device) * w
    sy = torch.rand(7, generator=g, device=device) * h
    lv = torch.tensor(LEVELS_C1, device=device, dtype=torch.float32)
    pick = torch.randint(0, 7, (7,), generator=g, device=device)
    base = lv[pick][_voronoi_labels(w, h, sx, sy)]
    noise = torch.randn((h, w), generator=g, device=device) * 8.0
    return _to_u8(base + noise)


def c2(seed: int = CONFIGS["C2"].seed, device="cpu", w: int = 5184, h: int = 3456,
       n_ellipses: int = 40) -> torch.Tensor:
    """Linear gradient 0-200 + filled rotated ellipses (offset +-60) + N(0, 5^2)."""
    g = _gen(seed, device)
    xs = torch.arange(w, device=device, dtype=torch.float32)
    ys = torch.arange(h, device=device, dtype=torch.float32)
    img = 100.0 * (xs[None, :] / max(w - 1, 1) + ys[:, None] / max(h - 1, 1))
    cx = torch.rand(n_ellipses, generator=g, device=device) * w
    cy = torch.rand(n_ellipses, generator=g, device=device) * h
    ax = 50.0 + torch.rand(n_ellipses, generator=g, device=device) * 550.0
    ay = 50.0 + torch.rand(n_ellipses, generator=g, device=device) * 550.0
    th = torch.rand(n_ellipses, generator=g, device=device) * torch.pi
    off = (torch.rand(n_ellipses, generator=g, device=device) * 2.0 - 1.0) * 60.0
    for i in range(n_ellipses):
        x0 = int(max(0, float(cx[i] - 610)))
        x1 = int(min(w, float(cx[i] + 610)))
        y0 = int(max(0, float(cy[i] - 610)))
        y1 = int(min(h, float(cy[i] + 610)))
        if x0 >= x1 or y0 >= y1:
            continue
        dx = xs[x0:x1][None, :] - cx[i]
        dy = ys[y0:y1][:, None] - cy[i]
        c, s = torch.cos(th[i]), torch.sin(th[i])
        u = (dx * c + dy * s) / ax[i]
        v = (-dx * s + dy * c) / ay[i]
        inside = (u * u + v * v) <= 1.0
        img[y0:y1, x0:x1] += inside.to(torch.float32) * off[i]
    img = img + torch.randn((h, w), generator=g, device=device) * 5.0
    return _to_u8(img)


def c3(seed: int = CONFIGS["C3"].seed, device="cpu", n: int = 512, w: int = 1920, h: int = 1080,
       regions: int = 12) -> torch.Tensor:
    """n frames: 12-region Voronoi whose seeds drift 2 px/frame, + N(0, 6^2)."""
    g = _gen(seed, device)
    sx = torch.rand(regions, generator=g, device=device) * w
    sy = torch.rand(regions, generator=g, device=device) * h
    ang = torch.rand(regions, generator=g, device=device) * 2 * torch.pi
    vx, vy = 2.0 * torch.cos(ang), 2.0 * torch.sin(ang)
    lv = torch.randint(0, 256, (regions,), generator=g, device=device).to(torch.float32)
    out = torch.empty((n, h, w), dtype=torch.uint8, device=device)
    for f in range(n):
        lab = _voronoi_labels(w, h, sx + vx * f, sy + vy * f)
        noise = torch.randn((h, w), generator=g, device=device) * 6.0
        out[f] = _to_u8(lv[lab] + noise)
    return out


def c4(seed: int = CONFIGS["C4"].seed, device="cpu", w: int = 16384, h: int = 16384) -> torch.Tensor:
    """i.i.d. uniform bytes."""
    g = _gen(seed, device)
    return torch.randint(0, 256, (h, w), generator=g, device=device, dtype=torch.uint8)


def c5(seed: int = CONFIGS["C5"].seed, device="cpu", n: int = 65536, size: int = 128,
       chunk: int = 4096) -> torch.Tensor:
    """Image i from family i mod 4: (a) 3-level {0,128,255} horizontal stripes
    of random width, (b) constant (empty boundary), (c) 0/255 checkerboard
    with cell 1-8 px, (d) bimodal N(60,15^2)/N(190,15^2) i.i.d., clipped."""
    g = _gen(seed, device)
    out = torch.empty((n, size, size), dtype=torch.uint8, device=device)
    ys = torch.arange(size, device=device)
    xs = torch.arange(size, device=device)
    lv3 = torch.tensor([0, 128, 255], device=device, dtype=torch.uint8)
    for s0 in range(0, n, chunk):
        m = min(chunk, n - s0)
        fam = (torch.arange(s0, s0 + m, device=device) % 4)
        # (a) stripes: a new stripe starts at row r with prob 1/12
        starts = torch.rand((m, size), generator=g, device=device) < (1.0 / 12.0)
        sid = torch.cumsum(starts.to(torch.int64), dim=1)
        first = torch.randint(0, 3, (m, 1), generator=g, device=device)
        stripes = lv3[(sid + first) % 3][:, :, None].expand(m, size, size)
        # (b) constant
        const = torch.randint(0, 256, (m, 1, 1), generator=g, device=device, dtype=torch.int64)
        const = const.to(torch.uint8).expand(m, size, size)
        # (c) checkerboard
        cell = torch.randint(1, 9, (m, 1, 1), generator=g, device=device)
        chk = (((ys[None, :, None] // cell) + (xs[None, None, :] // cell)) % 2).to(torch.uint8) * 255
        # (d) bimodal
        mode = torch.rand((m, size, size), generator=g, device=device) < 0.5
        mu = torch.where(mode, torch.tensor(60.0, device=device), torch.tensor(190.0, device=device))
        bim = _to_u8(mu + torch.randn((m, size, size), generator=g, device=device) * 15.0)
        f = fam[:, None, None]
        img = torch.where(f == 0, stripes, torch.where(f == 1, const, torch.where(f == 2, chk, bim)))
        out[s0:s0 + m] = img
    return out


def generate(name: str, device="cpu", **overrides) -> torch.Tensor:
    """Full-size input of config `name` as a (n, h, w) uint8 tensor."""
    cfg = CONFIGS[name]
    fn = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}[name]
    x = fn(cfg.seed, device, **overrides)
    return x if x.dim() == 3 else x[None]
