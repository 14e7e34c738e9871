"""NEXT-1: receding-horizon MPC on the batch solver.

P:585: "We also built an MPC on top of our batch optimizer, wherein we
warm-started the Lagrange multipliers lambda_l, lambda_psi,l with the solution
obtained at the previous control loop.  We ran the MPC with a time-budget of
0.04 s which was enough to perform 10 iterations of our optimizer with a batch
size of 1000."  Every control tick:

  1. boundary: the executed state (p, v, a of x, y, psi) at t = 0; at the end
     of the horizon the desired straight line (constant velocity
     v_des along +x), x = v_des (t_now + T_h), y = 0, zero heading and rates;
  2. samples: fresh STOMP-style Gaussian samples around the straight segment
     start -> goal ("always initialized with a Gaussian distribution
     ... centered around a straight-line trajectory"), drawn by the backend:
     bmc_sample_init on the device (NEXT-2: Philox stream (seed, tick)), the
     oracle sampler in the tests, synth.make_init for a backend without one;
  3. one batch solve of K iterations with lambda_in = the previous tick's
     lambda_out, instance by instance (kept on the device);
  4. execute dt of the best trajectory (argmin key, G17): the new state is the
     best trajectory's p, v, a at t = dt (Bernstein evaluation, host fp64 on
     the 55 coefficients read back).

Readings (G25-G27): the paper gives neither the MPC horizon nor
the tick length; `MPCConfig` defaults to a 10 s horizon, q = 100 samples and a
0.1 s tick.  The solver (GPU or, in tests, the oracle) is pluggable; the
control loop itself is host logic around the hot path.
"""
from __future__ import annotations

import ctypes as C
import functools

from dataclasses import dataclass, field
from math import comb
from typing import Callable, Optional

import numpy as np

from synth import Config, make_init, tracks_at

from .distributed import RECORD_WORDS, pack_record


@dataclass(frozen=True)
class MPCConfig:
    cfg: Config                 # q, m, n, bounds, weights of the solve (cfg.T is overridden by horizon)
    horizon: float = 10.0       # T_h, seconds (reading G25)
    dt: float = 0.1             # control tick, seconds (reading G26)
    K: int = 10                 # AM iterations per tick
    v_des: float = 1.0          # desired speed along +x
    sigma_x: float = 1.0        # STOMP sample spread (synth.make_init)
    sigma_y: float = 2.0
    seed: int = 0

    @property
    def solve_cfg(self) -> Config:
        return self.cfg.with_(T=self.horizon, K=self.K)


@functools.lru_cache(maxsize=16)   # constant per configuration: computed once, not per tick
def bernstein_rows(degree: int, tau: float, T: float) -> np.ndarray:
    """[3][degree+1]: B_k(tau), dB_k/dt, d2B_k/dt2 at tau = t / T (fp64)."""
    n = degree

    def b(d, k):
        return comb(d, k) * tau ** k * (1.0 - tau) ** (d - k) if 0 <= k <= d else 0.0

    out = np.zeros((3, n + 1))
    for k in range(n + 1):
        out[0, k] = b(n, k)
        out[1, k] = n * (b(n - 1, k - 1) - b(n - 1, k)) / T
        out[2, k] = n * (n - 1) * (b(n - 2, k - 2) - 2.0 * b(n - 2, k - 1) + b(n - 2, k)) / (T * T)
    out.flags.writeable = False   # shared by the cache
    return out


@dataclass
class TickResult:
    t: float
    state: np.ndarray           # [3][3] (x, y, psi) x (p, v, a) after the tick
    best: int
    coeffs: np.ndarray          # [5][11] best trajectory of this tick
    residual: np.ndarray        # [2] of the best
    cost: float
    solve_ms: float             # device time of the solve (GPU backend) or host time


class MPC:
    """Receding-horizon loop; `solve(init, obs_xy, obs_ab, bnd, K, lambda_in) -> dict` is the
    backend (GpuBackend below, or an oracle-backed callable in the tests)."""

    def __init__(self, mc: MPCConfig, tracks: dict, backend: Callable, B: int,
                 start: Optional[np.ndarray] = None):
        self.mc, self.tracks, self.backend, self.B = mc, tracks, backend, int(B)
        self.t = 0.0
        # state [x, y, psi] x [p, v, a]: at rest heading along +x, moving at v_des
        self.state = np.zeros((3, 3)) if start is None else np.array(start, dtype=np.float64)
        if start is None:
            self.state[0, 1] = mc.v_des
        self.lam = None             # backend-owned (device tensor for the GPU)
        self.tick_no = 0
        self.log: list[TickResult] = []

    def boundary(self) -> np.ndarray:
        mc = self.mc
        bnd = np.zeros((3, 6))
        bnd[:, 0:3] = self.state
        bnd[0, 3] = mc.v_des * (self.t + mc.horizon)
        bnd[0, 4] = mc.v_des
        return bnd

    def problem(self) -> dict:
        sc, mc = self.mc.solve_cfg, self.mc
        bnd = self.boundary()
        if hasattr(self.backend, "sample"):
            init = self.backend.sample(self.B, bnd, seed=mc.seed, stream=self.tick_no, sigma_x=mc.sigma_x,
                                       sigma_y=mc.sigma_y)
        else:
            init = make_init(sc, seed=mc.seed * 100003 + self.tick_no, B=self.B, sigma_x=mc.sigma_x,
                             sigma_y=mc.sigma_y, bnd=bnd)
        obs = tracks_at(self.tracks, self.t, sc.q, sc.T)
        ab = np.ascontiguousarray(self.tracks["ab"].astype(np.float32))
        return dict(init=init, obs_xy=obs, obs_ab=ab, bnd=bnd)

    def tick(self) -> TickResult:
        mc, sc = self.mc, self.mc.solve_cfg
        pr = self.problem()
        out = self.backend(pr["init"], pr["obs_xy"], pr["obs_ab"], pr["bnd"], mc.K, self.lam)
        self.lam = out["lambda_out"]
        best = int(out["best"])
        c = np.asarray(out["best_coeffs"], dtype=np.float64).reshape(5, sc.degree + 1)
        rows = bernstein_rows(sc.degree, mc.dt / sc.T, sc.T)
        # executed state at t = dt: position / velocity / acceleration of x (block 0),
        # y (block 2) and psi (block 4)
        self.state = np.stack([rows @ c[0], rows @ c[2], rows @ c[4]])
        self.t += mc.dt
        self.tick_no += 1
        r = TickResult(self.t, self.state.copy(), best, c, np.asarray(out["best_residual"]), float(out["best_cost"]),
                       float(out.get("solve_ms", 0.0)))
        self.log.append(r)
        return r


class GpuBackend:
    """bmc_solve on the device; lambda stays on the device between ticks, the best
    trajectory (55 floats) and its residual / cost are read back per tick."""

    def __init__(self, mc: MPCConfig, device: int = 0):
        import torch
        from .bmc import solver_for
        self.torch = torch
        self.dev = torch.device("cuda", device)
        self.solver = solver_for(mc.solve_cfg, device=device)
        self.out = None
        self.ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))

    def sample(self, B, bnd, seed, stream, sigma_x, sigma_y):
        """STOMP samples drawn on the device (bmc_sample_init, NEXT-2); stays on the device."""
        buf = getattr(self, "init_buf", None)
        if buf is not None and buf.shape[0] != B:
            buf = None
        self.init_buf = self.solver.sample_init(B, bnd, seed, stream, sigma_x=sigma_x, sigma_y=sigma_y, out=buf)
        return self.init_buf

    def _to_dev(self, key, a):
        """Host array -> device through a pinned staging buffer (asynchronous H2D)."""
        torch = self.torch
        if isinstance(a, torch.Tensor):
            return a
        a = np.ascontiguousarray(a, dtype=np.float32)
        st = self.stage.get(key)
        if st is None or st[0].shape != a.shape:
            st = (torch.empty(a.shape, dtype=torch.float32).pin_memory(),
                  torch.empty(a.shape, dtype=torch.float32, device=self.dev))
            self.stage[key] = st
        st[0].numpy()[...] = a
        st[1].copy_(st[0], non_blocking=True)
        return st[1]

    def __call__(self, init, obs_xy, obs_ab, bnd, K, lam):
        torch = self.torch
        if not hasattr(self, "stage"):
            self.stage = {}
        init_d, obs_d, ab_d = self._to_dev("init", init), self._to_dev("obs", obs_xy), self._to_dev("ab", obs_ab)
        B = init.shape[0]
        if self.out is None or self.out[0]["coeffs"].shape[0] != B:
            mk = lambda *s: torch.empty(s, dtype=torch.float32, device=self.dev)
            self.out = [dict(coeffs=mk(B, 5, 11), lambda_out=mk(B, 5, 11), residual=mk(B, 2), cost=mk(B),
                             best=torch.empty(2, dtype=torch.int64, device=self.dev)) for _ in range(2)]
            self.flip = 0
            # read-back of the best instance: bmc_pack_best gathers {key, 55 coefficients,
            # r1, r_psi, J} on the device into one 256-byte record, copied once per tick
            self.rec = torch.empty(RECORD_WORDS, dtype=torch.int64, device=self.dev)
            self.rb = torch.empty(RECORD_WORDS, dtype=torch.int64).pin_memory()
        o = self.out[self.flip]          # double-buffered: lambda_in of this tick is the other buffer
        self.flip ^= 1
        stream = torch.cuda.current_stream(self.dev)
        self.ev[0].record(stream)
        self.solver.solve(init_d, obs_d if obs_xy.shape[0] else None, ab_d if obs_xy.shape[0] else None, bnd, K,
                          lambda_in=lam, out=o)
        self.ev[1].record(stream)
        # one read-back per tick: the best instance's record, gathered by the library
        pack_record(o["best"], o["coeffs"], 0, self.rec, C.c_void_p(stream.cuda_stream), o["residual"], o["cost"])
        self.rb.copy_(self.rec, non_blocking=True)
        stream.synchronize()
        key = int(self.rb[0])
        rb = self.rb.numpy()[1:].view(np.float32)
        res = dict(lambda_out=o["lambda_out"], best=key & ((1 << 30) - 1), best_coeffs=rb[:55].copy(),
                   best_residual=rb[55:57].copy(), best_cost=float(rb[57]))
        res["solve_ms"] = self.ev[0].elapsed_time(self.ev[1])
        return res
