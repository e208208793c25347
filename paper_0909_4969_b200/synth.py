"""Seeded synthetic inputs with the BASELINE.json config shapes (no public
dataset is named; SURVEY.md §8d generator): Tucker core with N(0,1) entries
times column-orthonormal factors, plus Gaussian noise with
sigma = rho * |X0|_F / sqrt(numel).

numpy (CPU, small sizes, used by the parity tests so oracle and device see the
same bytes) and torch (device, the multi-GB bench tensors) versions.  The
torch version returns a flat first-mode-fastest CUDA buffer.
"""
from __future__ import annotations

import numpy as np

# name -> (dims, ranks, noise_rel, p, sweeps, dtype)
# C4 uses the tensor-stream generator: host factor diag(l) Q with
# l ~ lognormal(0, 1) (heavy-tailed host loads, not orthonormal), time factor
# = orthonormalised sin/cos harmonics of a 288-tick daily period.
KIND = {"c4": "stream"}
CONFIGS = {
    "c1": ((100, 12, 1024), (5, 5, 5), 0.01, 0.1, 3, "float64"),
    "c2": ((512, 512, 512), (10, 10, 10), 0.01, 0.05, 5, "float32"),
    "c3": ((128, 128, 64, 256), (8, 8, 8, 8), 0.02, 0.02, 5, "float32"),
    "c4": ((1000, 64, 65536), (10, 6, 20), 0.05, 0.01, 3, "float32"),
    "c5": ((1024, 1024, 1024), (16, 16, 16), 0.01, 0.1, 5, "float32"),
    # C5's sampling-rate sweep: p = 1 takes the dense route (tcgen05 Gram and
    # mode products), the others the sparse route
    "c5p1": ((1024, 1024, 1024), (16, 16, 16), 0.01, 1.0, 5, "float32"),
    "c5p01": ((1024, 1024, 1024), (16, 16, 16), 0.01, 0.01, 5, "float32"),
    "c5p001": ((1024, 1024, 1024), (16, 16, 16), 0.01, 0.001, 5, "float32"),
}


PERIOD = 288  # 5-minute buckets per day


def harmonics(n, r, period=PERIOD) -> np.ndarray:
    """n x r orthonormalised sin/cos harmonics of the daily period (time factor)."""
    t = np.arange(n, dtype=np.float64)[:, None]
    cols = []
    h = 1
    while len(cols) < r:
        w = 2.0 * np.pi * h * t / period
        cols += [np.sin(w), np.cos(w)]
        h += 1
    q, _ = np.linalg.qr(np.hstack(cols[:r]))
    return q


def stream_factors(dims, ranks, rng):
    """Factors of the tensor-stream generator (hosts x metrics x time)."""
    facs = []
    for m, (n, r) in enumerate(zip(dims, ranks)):
        if m == len(dims) - 1:
            facs.append(harmonics(n, r))
            continue
        q, _ = np.linalg.qr(rng.standard_normal((n, r)))
        if m == 0:
            q = np.exp(rng.standard_normal(n))[:, None] * q  # lognormal(0, 1) host loads
        facs.append(q)
    return facs


def lowrank_numpy(dims, ranks, noise_rel=0.01, seed=0, dtype=np.float64, kind=None) -> np.ndarray:
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(ranks)
    x = core
    if kind == "stream":
        facs = stream_factors(dims, ranks, rng)
    else:
        facs = [np.linalg.qr(rng.standard_normal((n, r)))[0] for n, r in zip(dims, ranks)]
    for m, q in enumerate(facs):
        x = np.moveaxis(np.tensordot(q, x, axes=([1], [m])), 0, m)
    if noise_rel > 0:
        sigma = noise_rel * np.sqrt((x * x).sum()) / np.sqrt(x.size)
        x = x + sigma * rng.standard_normal(x.shape)
    return np.asarray(x, dtype=dtype)


def lowrank_torch(dims, ranks, noise_rel=0.01, seed=0, dtype="float32", device="cuda", kind=None):
    """Flat first-mode-fastest CUDA tensor of the config (generated on device)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    d = len(dims)
    core = torch.randn(*ranks, generator=g, device=device, dtype=torch.float64)
    facs = []
    for m, (n, r) in enumerate(zip(dims, ranks)):
        if kind == "stream" and m == d - 1:
            facs.append(torch.as_tensor(harmonics(n, r), device=device))
            continue
        a = torch.randn(n, r, generator=g, device=device, dtype=torch.float64)
        q, _ = torch.linalg.qr(a)
        if kind == "stream" and m == 0:
            q = torch.exp(torch.randn(n, generator=g, device=device, dtype=torch.float64))[:, None] * q
        facs.append(q)
    # X0 in C order with reversed axes == first-mode-fastest flat buffer
    letters = "abcdefgh"[:d]
    ranks_l = "ABCDEFGH"[:d]
    spec = ranks_l + "," + ",".join(f"{letters[m]}{ranks_l[m]}" for m in range(d)) + "->" + letters[::-1]
    tdt = {"float32": torch.float32, "float64": torch.float64}[dtype]
    x0 = torch.einsum(spec, core, *facs)  # fp64, shape dims[::-1]
    norm = torch.linalg.vector_norm(x0)
    x = x0.to(tdt)
    del x0
    if noise_rel > 0:
        sigma = float(noise_rel * norm / np.sqrt(float(np.prod(dims))))
        x.add_(torch.randn(x.shape, generator=g, device=device, dtype=tdt), alpha=sigma)
    return x.reshape(-1)
