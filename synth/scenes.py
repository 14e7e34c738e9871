"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no basis matrix, no KKT, no
projection): it only draws obstacle tracks and initial Bernstein control
points, and names the configurations of BASELINE.json.  Both the CUDA path and
the oracle consume exactly these arrays (fp32, rounded once; the oracle promotes
them exactly to fp64).

Recipe (shaped like the paper's benchmarks P:587-589):
  * horizon T = 30 s ("around 30s"), q samples at t_k = k T / (q - 1);
  * robot: start (0, 0) at 1.0 m/s along +x, goal (30, 0) at 1.0 m/s, zero
    accelerations, heading 0 with zero rates;
  * footprint: m circles of radius 0.3 m on the heading axis, offsets
    m=1: {0}; m=2: {-0.3, 0.3}; m=3: {-0.5, 0, 0.5}; m=4: {+-0.25, +-0.75};
  * obstacles: humans of radius 0.3 m, inflated by the circle radius, so
    a = b = 0.6 m (P:97 one (a, b) for all obstacles);
  * static scenes: centres x ~ U(8, 22), y ~ U(-1, 1) (block the line);
  * dynamic scenes: x0 ~ U(3, 27), y0 ~ U(-4, 4), pairwise gap >= 1.2 m and
    >= 2 m from start/goal (rejection sampling); half "same direction"
    vx ~ U(0, 0.3), half "opposite" vx ~ U(-1.0, -0.3),
    vy ~ U(-0.1, 0.1); x_j(t_k) = x0 + v t_k (constant velocity);
  * initial samples (STOMP-style around the straight line): the
    degree-10 Bernstein control points of the straight line are the equally
    spaced points between start and goal; control points 3..7 (the ones that
    do not enter position, velocity or acceleration at either end) get smooth
    Gaussian noise N(0, s^2 (D^T D)^-1) with D the second-difference operator
    on the control polygon, s_x = 1 m, s_y = 5 m; instance 0 is the
    unperturbed line; c_psi = 0.  Generated in fp64, rounded to fp32 once.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Dict, List, Optional

import numpy as np

T_HORIZON = 30.0
DEGREE = 10
CIRCLE_RADIUS = 0.3
OBSTACLE_RADIUS = 0.3

OFFSETS = {
    1: [0.0],
    2: [-0.3, 0.3],
    3: [-0.5, 0.0, 0.5],
    4: [-0.75, -0.25, 0.25, 0.75],
}

# bnd[3][6]: x, y, psi  x  (p0, v0, a0, pT, vT, aT)
BND_STRAIGHT = np.array(
    [[0.0, 1.0, 0.0, 30.0, 1.0, 0.0], [0.0, 0.0, 0.0, 0.0, 0.0, 0.0], [0.0, 0.0, 0.0, 0.0, 0.0, 0.0]],
    dtype=np.float64,
)


@dataclass(frozen=True)
class Config:
    name: str
    B: int
    q: int
    m: int
    n: int
    K: int
    dynamic: bool
    v_max: float = 2.0
    a_max: float = 2.0
    rho: float = 1.0
    rho_psi: float = 1.0
    res_tol: float = 0.05
    T: float = T_HORIZON
    degree: int = DEGREE
    description: str = ""

    @property
    def offsets(self) -> List[float]:
        return list(OFFSETS[self.m]) if self.m in OFFSETS else list(np.linspace(-0.75, 0.75, self.m))

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS: Dict[str, Config] = {
    "C1": Config("C1", B=8, q=50, m=2, n=4, K=50, dynamic=False,
                 description="batch 8, horizon 50, 2 circles, 4 static obstacles, 50 iterations"),
    "C2": Config("C2", B=100, q=100, m=3, n=10, K=100, dynamic=True,
                 description="batch 100, horizon 100, 3 circles, 10 dynamic obstacles, 100 iterations"),
    "C3": Config("C3", B=1000, q=100, m=3, n=30, K=100, dynamic=True,
                 description="batch 1000 Gaussian inits, horizon 100, 3 circles, 30 dynamic obstacles, 100 iterations"),
    "C4": Config("C4", B=1000, q=100, m=4, n=50, K=200, dynamic=True, v_max=1.2, a_max=0.5,
                 description="batch 1000, horizon 100, 4 circles, 50 dynamic obstacles, tight v/a bounds, 200 iterations"),
    "C5": Config("C5", B=16384, q=100, m=3, n=30, K=100, dynamic=True,
                 description="batch scaling sweep 100-16384, horizon 100, 3 circles, 30 obstacles"),
}


def time_grid(q: int, T: float = T_HORIZON) -> np.ndarray:
    return np.arange(q, dtype=np.float64) * (T / (q - 1))


def _static_obstacles(rng, n: int):
    x0 = rng.uniform(8.0, 22.0, size=n)
    y0 = rng.uniform(-1.0, 1.0, size=n)
    return x0, y0, np.zeros(n), np.zeros(n)


def _dynamic_obstacles(rng, n: int):
    xs: List[float] = []
    ys: List[float] = []
    tries = 0
    while len(xs) < n:
        tries += 1
        x = rng.uniform(3.0, 27.0)
        y = rng.uniform(-4.0, 4.0)
        gap = 1.2 if tries < 20000 else 0.0
        if np.hypot(x, y) < 2.0 or np.hypot(x - 30.0, y) < 2.0:
            continue
        if any(np.hypot(x - a, y - b) < gap for a, b in zip(xs, ys)):
            continue
        xs.append(x)
        ys.append(y)
    n_same = n // 2
    vx = np.concatenate([rng.uniform(0.0, 0.3, size=n_same), rng.uniform(-1.0, -0.3, size=n - n_same)])
    vy = rng.uniform(-0.1, 0.1, size=n)
    return np.array(xs), np.array(ys), vx, vy


def make_scene(cfg: Config, seed: int = 0, ab: Optional[np.ndarray] = None) -> dict:
    """Obstacle tracks obs_xy [n][2][q] fp32, semi-axes obs_ab [n][2] fp32, bnd [3][6] fp64."""
    rng = np.random.default_rng(seed)
    n, q = cfg.n, cfg.q
    t = time_grid(q, cfg.T)
    if n > 0:
        x0, y0, vx, vy = (_dynamic_obstacles if cfg.dynamic else _static_obstacles)(rng, n)
        obs = np.empty((n, 2, q), dtype=np.float64)
        obs[:, 0, :] = x0[:, None] + vx[:, None] * t[None, :]
        obs[:, 1, :] = y0[:, None] + vy[:, None] * t[None, :]
    else:
        obs = np.zeros((0, 2, q))
    if ab is None:
        ab = np.full((n, 2), CIRCLE_RADIUS + OBSTACLE_RADIUS)
    return dict(
        obs_xy=np.ascontiguousarray(obs.astype(np.float32)),
        obs_ab=np.ascontiguousarray(np.asarray(ab, dtype=np.float64).reshape(n, 2).astype(np.float32)),
        bnd=BND_STRAIGHT.copy(),
    )


def make_tracks(cfg: Config, seed: int = 0) -> dict:
    """The obstacle motions of `make_scene` as constant-velocity tracks
    (x0, y0, vx, vy [n] fp64, semi-axes ab [n][2]) for receding-horizon use."""
    rng = np.random.default_rng(seed)
    n = cfg.n
    if n > 0:
        x0, y0, vx, vy = (_dynamic_obstacles if cfg.dynamic else _static_obstacles)(rng, n)
    else:
        x0 = y0 = vx = vy = np.zeros(0)
    return dict(x0=x0, y0=y0, vx=vx, vy=vy, ab=np.full((n, 2), CIRCLE_RADIUS + OBSTACLE_RADIUS))


def tracks_at(tracks: dict, t0: float, q: int, T: float) -> np.ndarray:
    """Obstacle positions obs_xy [n][2][q] fp32 at absolute times t0 + t_k."""
    t = t0 + time_grid(q, T)
    obs = np.empty((tracks["x0"].size, 2, q), dtype=np.float64)
    obs[:, 0, :] = tracks["x0"][:, None] + tracks["vx"][:, None] * t[None, :]
    obs[:, 1, :] = tracks["y0"][:, None] + tracks["vy"][:, None] * t[None, :]
    return np.ascontiguousarray(obs.astype(np.float32))


def scene_blocker(q: int = 100, x: float = 15.0, a: float = 1.5) -> dict:
    """NEXT-3 (Fig. 1c): one static obstacle of semi-axes a on the straight
    start -> goal line; the batch should find both homotopy classes (above / below)."""
    obs = np.zeros((1, 2, q))
    obs[0, 0, :] = x
    return dict(obs_xy=obs.astype(np.float32), obs_ab=np.full((1, 2), a, np.float32), bnd=BND_STRAIGHT.copy())


def scene_wall_gap(q: int = 100, x: float = 15.0, gap: float = 1.2, half_width: float = 3.6,
                   human: float = OBSTACLE_RADIUS, inflate: float = CIRCLE_RADIUS) -> dict:
    """NEXT-3 (Table II trend): a wall of humans (radius `human`, centre spacing
    2 human) across the line at x, with a free gap of width `gap` centred on y = 0.  Obstacles
    are inflated by `inflate` (the footprint circle radius: 0.3 m for the multi-circle robot,
    0.8 m for the single disk that covers the same 1.6 x 0.6 m footprint)."""
    edge = gap / 2 + human
    ys = []
    y = edge
    while y <= half_width:
        ys += [y, -y]
        y += 2 * human
    n = len(ys)
    obs = np.zeros((n, 2, q))
    obs[:, 0, :] = x
    obs[:, 1, :] = np.array(ys)[:, None]
    return dict(obs_xy=obs.astype(np.float32), obs_ab=np.full((n, 2), human + inflate, np.float32),
                bnd=BND_STRAIGHT.copy())


def line_control_points(bnd: np.ndarray = BND_STRAIGHT, degree: int = DEGREE) -> np.ndarray:
    """Control points [2][degree+1] of the constant-velocity segment start->goal."""
    s = np.arange(degree + 1) / degree
    x = bnd[0, 0] + (bnd[0, 3] - bnd[0, 0]) * s
    y = bnd[1, 0] + (bnd[1, 3] - bnd[1, 0]) * s
    return np.stack([x, y])


def _smooth_cov(degree: int) -> np.ndarray:
    nv = degree + 1
    D = np.zeros((nv - 2, nv))
    for i in range(nv - 2):
        D[i, i:i + 3] = [1.0, -2.0, 1.0]
    R = D.T @ D
    free = np.arange(3, nv - 3)
    cov = np.linalg.inv(R[np.ix_(free, free)])
    return cov / np.max(np.diag(cov))


def make_init(cfg: Config, seed: int = 1000, B: Optional[int] = None, sigma_x: float = 1.0,
              sigma_y: float = 5.0, bnd: np.ndarray = BND_STRAIGHT) -> np.ndarray:
    """Initial samples init [B][3][nv] fp32: (c_x, c_y, c_psi)."""
    B = cfg.B if B is None else B
    nv = cfg.degree + 1
    rng = np.random.default_rng(seed)
    base = line_control_points(bnd, cfg.degree)
    L = np.linalg.cholesky(_smooth_cov(cfg.degree))
    free = np.arange(3, nv - 3)
    out = np.zeros((B, 3, nv))
    out[:, 0, :] = base[0]
    out[:, 1, :] = base[1]
    if B > 1:
        zx = rng.standard_normal((B - 1, free.size))
        zy = rng.standard_normal((B - 1, free.size))
        out[1:, 0, free] += sigma_x * zx @ L.T
        out[1:, 1, free] += sigma_y * zy @ L.T
    return np.ascontiguousarray(out.astype(np.float32))


def make_problem(cfg: Config, scene_seed: int = 0, B: Optional[int] = None, init_seed: Optional[int] = None):
    """Scene + initial samples for one configuration (the recipe above)."""
    sc = make_scene(cfg, scene_seed)
    init = make_init(cfg, 1000 + scene_seed if init_seed is None else init_seed, B=B)
    sc["init"] = init
    return sc
