"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NONE of the method's arithmetic (no hashing, sampling,
graph construction, partitioning or layer math): it only draws point clouds,
node fields, latent features, weights and upstream gradients with numpy's
PCG64, so that the CUDA path and the CPU oracle receive identical arrays.
The recipe for every config is stated in DESIGN.md §"Input recipe"
(BASELINE.json configs).
"""
from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 20240223
SEED_GEOMETRY, SEED_FIELDS, SEED_SAMPLING, SEED_CAPPING = 1, 2, 3, 4
SEED_FEATURES, SEED_WEIGHTS, SEED_GRAD = 5, 6, 7


@dataclass
class Config:
    name: str
    kind: str               # darcy | airfoil | step | weak
    P: int                  # sub-domains
    r: float                # kernel radius
    n_e: int                # edge cap
    d: int                  # latent width (d_in = d_out)
    k: int                  # kappa_phi hidden width
    L: int                  # layers (hops)
    s: int = 0              # sampled nodes (0 -> all)
    grid: int = 0           # darcy grid side
    n_points: int = 0       # point-cloud size
    edge_mode: str = "concat"
    extra: dict = field(default_factory=dict)

    @property
    def dim(self):
        return 3 if self.kind in ("step", "weak") else 2


CONFIGS = {
    # BASELINE.json configs[0]
    "tiny": Config("tiny", "darcy", P=1, r=0.25, n_e=64, d=16, k=32, L=2, s=64, grid=16,
                   edge_mode="diff"),
    # configs[1]: Darcy 241^2, 4 sub-domains x 4096 sampled nodes, width 64, 6 layers
    "darcy": Config("darcy", "darcy", P=4, r=0.2, n_e=64, d=64, k=256, L=6, s=16384, grid=241,
                    edge_mode="diff"),
    # configs[2]: 2-D airfoil ~2e5 nodes, 8 sub-domains, edge attr (x_i,x_j,a_i,a_j), width 64
    "airfoil": Config("airfoil", "airfoil", P=8, r=0.05, n_e=64, d=64, k=256, L=4,
                      n_points=200_000),
    # configs[3]: 3-D step ~1.6e5 nodes, ~1e7 edges, 8 sub-domains, width 32
    "step": Config("step", "step", P=8, r=0.0888, n_e=64, d=32, k=256, L=4, n_points=163_840),
    # configs[4]: weak scaling, ~2M edges per GPU (P filled in at run time)
    "weak": Config("weak", "weak", P=1, r=0.0956, n_e=64, d=32, k=256, L=4,
                   extra=dict(per_part=32_768)),
}


def rng(offset: int, salt: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([BASE_SEED + offset, salt]))


# ---------------------------------------------------------------- geometry ---

def darcy_points(n: int):
    """n x n grid on [0,1]^2 (reading R20: x = fl32(col/(n-1)), gid = row*n+col)
    with a thresholded Gaussian random field a in {3, 12}, z-scored."""
    t = (np.arange(n, dtype=np.float64) / (n - 1)).astype(np.float32)
    yy, xx = np.meshgrid(t, t, indexing="ij")
    coords = np.stack([xx.ravel(), yy.ravel()], axis=1).astype(np.float32)
    g = rng(SEED_FIELDS)
    noise = g.standard_normal((n, n))
    f = np.fft.fft2(noise)
    kx = np.fft.fftfreq(n) * n
    kk = np.sqrt(kx[:, None] ** 2 + kx[None, :] ** 2)
    f[kk > 8] = 0.0
    field_ = np.real(np.fft.ifft2(f))
    a = np.where(field_ >= 0.0, 12.0, 3.0)
    a = (a - a.mean()) / (a.std() + 1e-12)
    return coords, a.reshape(-1, 1).astype(np.float32)


def _naca0012(alpha_deg=5.0, m=2000):
    xs = 0.5 * (1 - np.cos(np.linspace(0, np.pi, m)))
    yt = 0.6 * (0.2969 * np.sqrt(xs) - 0.1260 * xs - 0.3516 * xs ** 2 + 0.2843 * xs ** 3
                - 0.1015 * xs ** 4)
    up = np.stack([xs, yt], 1)
    lo = np.stack([xs[::-1], -yt[::-1]], 1)
    poly = np.concatenate([up, lo[1:]], 0)
    a = np.deg2rad(-alpha_deg)
    c, s = np.cos(a), np.sin(a)
    p = poly - np.array([0.25, 0.0])
    p = np.stack([c * p[:, 0] - s * p[:, 1], s * p[:, 0] + c * p[:, 1]], 1) + np.array([0.25, 0.0])
    return p


def _inside_naca(pts, alpha_deg):
    """Analytic inside test: rotate back to the chord frame, |y'| < yt(x')."""
    a = np.deg2rad(alpha_deg)
    p = pts - np.array([0.25, 0.0])
    c, s = np.cos(a), np.sin(a)
    xr = c * p[:, 0] - s * p[:, 1] + 0.25
    yr = s * p[:, 0] + c * p[:, 1]
    xc = np.clip(xr, 0.0, 1.0)
    yt = 0.6 * (0.2969 * np.sqrt(xc) - 0.1260 * xc - 0.3516 * xc ** 2 + 0.2843 * xc ** 3
                - 0.1015 * xc ** 4)
    return (xr >= 0.0) & (xr <= 1.0) & (np.abs(yr) < yt)


def airfoil_points(n_points=200_000, alpha_deg=5.0):
    """NACA-0012 at alpha in [-2,4]x[-1.5,1.5]: 40% boundary-layer points offset
    along the normal by Exp(0.02), 60% uniform; a = (sdf, x cos a + y sin a)."""
    from scipy.spatial import cKDTree
    g = rng(SEED_GEOMETRY, 2)
    poly = _naca0012(alpha_deg)
    seg = np.diff(poly, axis=0)
    seglen = np.linalg.norm(seg, axis=1)
    cum = np.concatenate([[0], np.cumsum(seglen)])
    n_bl = int(0.4 * n_points)
    pts = []
    need = n_bl
    while need > 0:
        u = g.uniform(0, cum[-1], 2 * need)
        k = np.clip(np.searchsorted(cum, u) - 1, 0, len(seg) - 1)
        t = (u - cum[k]) / seglen[k]
        base = poly[k] + seg[k] * t[:, None]
        nrm = np.stack([seg[k, 1], -seg[k, 0]], 1) / seglen[k][:, None]
        off = g.exponential(0.02, len(u))
        cand = base + nrm * off[:, None]
        ok = ~_inside_naca(cand, alpha_deg)
        cand = cand[ok][:need]
        pts.append(cand)
        need -= len(cand)
    need = n_points - n_bl
    while need > 0:
        cand = np.stack([g.uniform(-2, 4, 2 * need), g.uniform(-1.5, 1.5, 2 * need)], 1)
        cand = cand[~_inside_naca(cand, alpha_deg)][:need]
        pts.append(cand)
        need -= len(cand)
    P = np.concatenate(pts, 0)
    tree = cKDTree(poly)
    dist, _ = tree.query(P)
    al = np.deg2rad(alpha_deg)
    a = np.stack([dist, P[:, 0] * np.cos(al) + P[:, 1] * np.sin(al)], 1)
    a = (a - a.mean(0)) / a.std(0)
    return P.astype(np.float32), a.astype(np.float32)


def step_points(n_points: int, length: float = 4.25, salt: int = 3):
    """Channel [0,length]x[0,1]x[0,1] minus the step block [0,0.5]x[0,0.5]x[0,1],
    uniform points; a = (u, v, w) analytic channel-like field."""
    g = rng(SEED_GEOMETRY, salt)
    out = []
    need = n_points
    while need > 0:
        c = np.stack([g.uniform(0, length, 2 * need), g.uniform(0, 1, 2 * need),
                      g.uniform(0, 1, 2 * need)], 1)
        ok = ~((c[:, 0] < 0.5) & (c[:, 1] < 0.5))
        c = c[ok][:need]
        out.append(c)
        need -= len(c)
    X = np.concatenate(out, 0)
    x, y, z = X[:, 0], X[:, 1], X[:, 2]
    u = 16 * y * (1 - y) * z * (1 - z)
    v = 0.1 * np.sin(2 * np.pi * x) * np.sin(np.pi * y)
    w = 0.1 * np.sin(np.pi * z) * np.cos(2 * np.pi * x)
    return X.astype(np.float32), np.stack([u, v, w], 1).astype(np.float32)


def points(cfg: Config, parts: int = None):
    """(coords float32 [N x dim], attr float32 [N x n_attr]) for a config."""
    if cfg.kind == "darcy":
        return darcy_points(cfg.grid)
    if cfg.kind == "airfoil":
        return airfoil_points(cfg.n_points)
    if cfg.kind == "step":
        return step_points(cfg.n_points)
    if cfg.kind == "weak":
        P = parts or cfg.P
        return step_points(cfg.extra["per_part"] * P, length=P + 0.25, salt=4)
    raise ValueError(cfg.kind)


def edge_dim(cfg: Config) -> int:
    n_attr = {"darcy": 1, "airfoil": 2, "step": 3, "weak": 3}[cfg.kind]
    if cfg.edge_mode == "diff":
        return cfg.dim + n_attr
    return 2 * (cfg.dim + n_attr)


# ----------------------------------------------------------- layer inputs ---

def node_features(n: int, d: int, salt: int = 0) -> np.ndarray:
    return rng(SEED_FEATURES, salt).standard_normal((n, d)).astype(np.float32)


def upstream_grad(n: int, d: int, salt: int = 0) -> np.ndarray:
    return rng(SEED_GRAD, salt).standard_normal((n, d)).astype(np.float32)


def weights(d_e: int, d_in: int, d_out: int, k: int, salt: int = 0) -> dict:
    """PyTorch-Linear-default uniform init U(+-1/sqrt(fan_in)); the last kappa
    layer is additionally scaled by 1/sqrt(d_in) so ||K^T v|| ~ ||v||."""
    g = rng(SEED_WEIGHTS, salt)

    def U(shape, fan_in, scale=1.0):
        b = 1.0 / np.sqrt(fan_in)
        return (g.uniform(-b, b, shape) * scale).astype(np.float32)

    return dict(
        W1=U((k, d_e), d_e), b1=U((k,), d_e),
        W2=U((k, k), k), b2=U((k,), k),
        W3=U((d_in * d_out, k), k, 1 / np.sqrt(d_in)), b3=U((d_in * d_out,), k, 1 / np.sqrt(d_in)),
        W_root=U((d_out, d_in), d_in), b=U((d_out,), d_in),
    )


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to bf16 (RNE) and return them widened to fp32.
    (Input preparation for the bf16 mode; not method arithmetic.)"""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = ((u + 0x7FFF + lsb) >> 16) << 16
    out = (u & 0xFFFFFFFF).astype(np.uint32).view(np.float32)
    nan = np.isnan(x)
    out = np.where(nan, x, out)
    return out.astype(np.float32)
