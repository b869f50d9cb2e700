"""Seeded synthetic fields shaped like the paper's scientific datasets (BASELINE.json ``configs``).

This module holds ONLY input generation -- none of the compressor's arithmetic -- so it may serve
both the oracle (tests) and the CUDA path (tests, bench).  The paper's datasets (Table 3, PAPER.md
P:857-886: Hurricane 100x500x500, NYX 512^3, Miranda 256x384x384, ...) are not available; these
fields stand in for them with the shapes and value structure named in BASELINE.json (recipe in
DESIGN.md "Input recipe").

Every field is a deterministic function of (config, shape, device): torch's CPU and CUDA generators
draw different streams, so a test always feeds the *same bytes* to both sides rather than
regenerating per side.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

__all__ = ["CONFIGS", "FieldConfig", "make_field", "grf", "config_by_name"]


@dataclass(frozen=True)
class FieldConfig:
    name: str
    shape: tuple
    dtype: torch.dtype
    seed: int
    eb: float            # error bound, value-range relative
    eb_mode: str         # "rel" or "abs"
    radius: int
    kind: str            # generator recipe
    desc: str


# BASELINE.json configs[0..4]; eb is value-range relative everywhere (REL); R=32768
CONFIGS = [
    FieldConfig("c1", (64, 64, 64), torch.float32, 0, 1e-3, "rel", 32768, "modes",
                "sum of 8 random sinusoidal modes + U(+-1e-3) noise"),
    FieldConfig("c2", (100, 500, 500), torch.float32, 1, 1e-4, "rel", 32768, "grf3_noise",
                "k^-3 Gaussian random field, unit variance, + N(0, sigma=1e-4) noise (Hurricane shape)"),
    FieldConfig("c3", (512, 512, 512), torch.float32, 2, 1e-3, "rel", 32768, "lognormal",
                "exp(2 G), G a unit-variance k^-2.5 GRF (NYX shape)"),
    FieldConfig("c4", (256, 384, 384), torch.float64, 3, 1e-6, "rel", 32768, "bumps",
                "32 anisotropic Gaussian bumps (width 10-60) + linear ramp, fp64 (Miranda shape)"),
    FieldConfig("c5", (1024, 2048, 2048), torch.float32, 4, 1e-3, "rel", 32768, "grf3",
                "k^-3 Gaussian random field, 16 GiB, sharded as block-aligned slabs"),
]


def config_by_name(name: str) -> FieldConfig:
    for c in CONFIGS:
        if c.name == name:
            return c
    raise KeyError(name)


def _wavenumbers(n: int, device, real_last: bool = False) -> torch.Tensor:
    # integer wavenumbers of a periodic box (numpy.fft.fftfreq(n) * n)
    if real_last:
        return torch.arange(n // 2 + 1, device=device, dtype=torch.float32)
    return torch.fft.fftfreq(n, d=1.0 / n, device=device).to(torch.float32)


@torch.no_grad()
def grf(shape, alpha: float, seed: int, device="cpu", chunk: int = 32) -> torch.Tensor:
    """Unit-variance Gaussian random field with power spectrum |k|^-alpha (float32).

    White N(0,1) noise -> rfftn -> multiply by |k|^(-alpha/2) (k=0 zeroed) -> irfftn -> normalise to
    mean 0, variance 1.  The spectral multiply and the moments run in chunks along dim 0 so the
    16 GiB config-5 field fits on one GPU beside its half spectrum.
    """
    n0, n1, n2 = shape
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
    spec = torch.fft.rfftn(x)
    del x
    k0 = _wavenumbers(n0, device)
    k1 = _wavenumbers(n1, device).view(1, n1, 1)
    k2 = _wavenumbers(n2, device, real_last=True).view(1, 1, n2 // 2 + 1)
    k12 = k1 * k1 + k2 * k2
    for s in range(0, n0, chunk):
        e = min(n0, s + chunk)
        kk = k0[s:e].view(-1, 1, 1) ** 2 + k12
        amp = torch.where(kk > 0, kk.clamp_min(1e-30) ** (-alpha / 4.0), torch.zeros_like(kk))
        spec[s:e] *= amp
        del kk, amp
    out = torch.fft.irfftn(spec, s=shape)
    del spec
    s1 = torch.zeros((), dtype=torch.float64, device=device)
    s2 = torch.zeros((), dtype=torch.float64, device=device)
    for s in range(0, n0, chunk):
        blk = out[s:s + chunk].to(torch.float64)
        s1 += blk.sum()
        s2 += (blk * blk).sum()
        del blk
    N = float(n0 * n1 * n2)
    mean = (s1 / N).item()
    var = (s2 / N).item() - mean * mean
    std = math.sqrt(max(var, 1e-300))
    out.sub_(mean).div_(std)
    return out


@torch.no_grad()
def _modes(shape, seed, device):
    n0, n1, n2 = shape
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    freq = torch.randint(1, 7, (8, 3), generator=g)
    phase = torch.rand(8, generator=g, dtype=torch.float64) * (2 * math.pi)
    i = torch.arange(n0, device=device, dtype=torch.float64).view(-1, 1, 1) / n0
    j = torch.arange(n1, device=device, dtype=torch.float64).view(1, -1, 1) / n1
    k = torch.arange(n2, device=device, dtype=torch.float64).view(1, 1, -1) / n2
    f = torch.zeros(shape, dtype=torch.float64, device=device)
    for m in range(8):
        a, b, c = (float(v) for v in freq[m])
        f += torch.sin(2 * math.pi * (a * i + b * j + c * k) + float(phase[m]))
    gd = torch.Generator(device=device)
    gd.manual_seed(seed + 1000)
    f += (torch.rand(shape, generator=gd, device=device, dtype=torch.float64) * 2 - 1) * 1e-3
    return f


@torch.no_grad()
def _bumps(shape, seed, device):
    n0, n1, n2 = shape
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    centres = torch.rand(32, 3, generator=g, dtype=torch.float64) * torch.tensor([n0, n1, n2], dtype=torch.float64)
    widths = 10 + torch.rand(32, 3, generator=g, dtype=torch.float64) * 50
    amps = torch.rand(32, generator=g, dtype=torch.float64) * 2 - 1
    i = torch.arange(n0, device=device, dtype=torch.float64).view(-1, 1, 1)
    j = torch.arange(n1, device=device, dtype=torch.float64).view(1, -1, 1)
    k = torch.arange(n2, device=device, dtype=torch.float64).view(1, 1, -1)
    f = i / n0 + j / n1 + k / n2
    for m in range(32):
        c, s = centres[m], widths[m]
        gi = torch.exp(-0.5 * ((i - float(c[0])) / float(s[0])) ** 2)
        gj = torch.exp(-0.5 * ((j - float(c[1])) / float(s[1])) ** 2)
        gk = torch.exp(-0.5 * ((k - float(c[2])) / float(s[2])) ** 2)
        f += float(amps[m]) * (gi * gj * gk)
    return f


@torch.no_grad()
def make_field(cfg: FieldConfig | str, device="cpu", shape=None) -> torch.Tensor:
    """Generate config ``cfg`` (optionally at another ``shape``, same recipe) on ``device``."""
    if isinstance(cfg, str):
        cfg = config_by_name(cfg)
    shape = tuple(shape or cfg.shape)
    if cfg.kind == "modes":
        f = _modes(shape, cfg.seed, device)
    elif cfg.kind == "grf3_noise":
        f = grf(shape, 3.0, cfg.seed, device)
        gd = torch.Generator(device=device)
        gd.manual_seed(cfg.seed + 1000)
        f += torch.randn(shape, generator=gd, device=device, dtype=torch.float32) * 1e-4
    elif cfg.kind == "lognormal":
        f = grf(shape, 2.5, cfg.seed, device)
        f.mul_(2.0).exp_()
    elif cfg.kind == "bumps":
        f = _bumps(shape, cfg.seed, device)
    elif cfg.kind == "grf3":
        f = grf(shape, 3.0, cfg.seed, device)
    else:
        raise ValueError(cfg.kind)
    return f.to(cfg.dtype).contiguous()
