"""Row f4: model-guided sparsity targeting -- the Guided Sparsity Learning (GSL) controller of
PAPER.md Sec. 2.3 (algorithm table, :489-510), driven by the B200 roofline model (libskc's
skc_model_* calls) instead of a CPU profile.

    Input:      pruning layer set S, performance model M
    Initialize: project speedup for each layer L in S using M; exclude all Ls without
                speedup potential from S
    Repeat:     train while actively pruning only Ls in S; periodically, for each L in S:
                  if sparsity >= upper bound of the useful range  -> stop pruning L
                  if stabilized sparsity <= lower bound           -> stop pruning L and
                                                                     restore its dense weights
    Until:      maximum iterations or convergence

In density x = 1 - sparsity (R9): "sparsity >= upper bound" is x <= x_lo (the
bandwidth crossover, no further speedup below it) and "sparsity <= lower bound" is
x >= x_hi = 1/alpha (sparse slower than dense).  Readings (R17): "stabilized" =
the density moved less than `eps` over the last `window` checks; a manual exclude list
covers layers the paper excludes for achievable-sparsity reasons the model cannot see
(conv1).  Training itself is out of scope: the controller is pure and is
driven by replayed density trajectories; applying its directives is the trainer's job.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import skc

EXCLUDED, ACTIVE, STOPPED_SATURATED, RESTORED_DENSE = ("EXCLUDED", "ACTIVE",
                                                       "STOPPED_SATURATED", "RESTORED_DENSE")
CONTINUE, STOP_PRUNING, RESTORE_DENSE = "CONTINUE", "STOP_PRUNING", "RESTORE_DENSE"


@dataclass(frozen=True)
class Platform:
    """F: dense FLOP/s, B: bytes/s, alpha: sparse compute overhead, beta: storage overhead."""
    name: str
    F: float
    B: float
    alpha: float
    beta: float = 2.0


# The paper's CPUs (Table 1; alpha PAPER.md:399-401, :471).
BDW = Platform("Xeon E5-2697 v4", 2.15e12, 1.22e11, 3.0)
ATOM = Platform("Atom C2750", 6.2e10, 1.5e10, 1.2)


def b200_platform(F_sgemm: float, B_hbm: float, sparse_rate: float) -> Platform:
    """B200 profile by the paper's method: alpha = F / the measured sparse
    rate (actual FLOP/s) where the layer is compute bound."""
    return Platform("B200", F_sgemm, B_hbm, F_sgemm / sparse_rate)


@dataclass
class LayerState:
    name: str
    geom: dict                      # K, C, R, S, H, W, stride, pad, groups
    cost: dict                      # skc_model_layer_cost (per image)
    window: dict                    # skc_model_window
    status: str
    trajectory: list = field(default_factory=list)   # (iteration, density)


@dataclass
class GslConfig:
    window: int = 3        # checks a density must be stable over
    eps: float = 0.01      # max density change that still counts as stable
    exclude: tuple = ()    # manual excludes (e.g. conv1)


class GslController:
    def __init__(self, layers: dict, platform: Platform, config: GslConfig = GslConfig(),
                 layer_platforms: dict = None):
        """layers: name -> geometry dict (K, C, R, S, H, W, stride, pad, groups).
        layer_platforms: optional name -> Platform measured for that layer (its own F and
        alpha: on B200 the dense rate and the sparse kernel's efficiency differ per layer
        shape); layers without one use `platform`."""
        if not layers:
            raise ValueError("GSL needs at least one layer")
        self.platform, self.config = platform, config
        self.layer_platforms = dict(layer_platforms or {})
        unknown = set(self.layer_platforms) - set(layers)
        if unknown:
            raise KeyError(f"platforms for unknown layers {sorted(unknown)}")
        self.layers = {}
        for name, g in layers.items():
            p = self.platform_of(name)
            cost = skc.skc_model_layer_cost(g["K"], g["C"], g["R"], g["S"], g["H"], g["W"],
                                            g.get("stride", 1), g.get("pad", 0),
                                            g.get("groups", 1), batch=1)
            win = skc.skc_model_window(cost, p.F, p.B, p.alpha, p.beta)
            ok = win["has_speedup_potential"] and name not in config.exclude
            self.layers[name] = LayerState(name, dict(g), cost, win, ACTIVE if ok else EXCLUDED)

    def platform_of(self, name: str) -> Platform:
        return self.layer_platforms.get(name, self.platform)

    def step(self, iteration: int, densities: dict) -> dict:
        """One periodic check; densities: name -> current density x of ACTIVE layers.
        Returns name -> directive for every ACTIVE layer (nothing for the others)."""
        out = {}
        for name, x in densities.items():
            if name not in self.layers:
                raise KeyError(f"unknown layer {name}")
            L = self.layers[name]
            if L.status != ACTIVE:
                continue
            L.trajectory.append((iteration, float(x)))
            w = self.config.window
            recent = [d for _, d in L.trajectory[-w:]]
            stable = len(recent) >= w and max(recent) - min(recent) < self.config.eps
            if x <= L.window["x_lo"]:
                L.status, out[name] = STOPPED_SATURATED, STOP_PRUNING
            elif stable and x >= L.window["x_hi"]:
                L.status, out[name] = RESTORED_DENSE, RESTORE_DENSE
            else:
                out[name] = CONTINUE
        return out

    def final_density(self, name: str) -> float:
        L = self.layers[name]
        if L.status in (EXCLUDED, RESTORED_DENSE) or not L.trajectory:
            return 1.0
        return L.trajectory[-1][1]

    def report(self) -> dict:
        """Per-layer status, final density, window and projected speedup; whole-net speedup =
        sum of dense times / sum of projected times (dense layers at dense time)."""
        rows, t_dense, t_net = [], 0.0, 0.0
        for name, L in self.layers.items():
            p = self.platform_of(name)
            x = self.final_density(name)
            pr = skc.skc_model_project(L.cost, x, p.F, p.B, p.alpha, p.beta)
            sparse = L.status in (ACTIVE, STOPPED_SATURATED)
            t = pr["t_sparse"] if sparse else pr["t_dense"]
            t_dense += pr["t_dense"]
            t_net += t
            rows.append(dict(layer=name, status=L.status, final_density=x,
                             x_lo=L.window["x_lo"], x_hi=L.window["x_hi"], alpha=p.alpha,
                             projected_speedup=pr["t_dense"] / t))
        return dict(platform=self.platform.name, alpha=self.platform.alpha, layers=rows,
                    net_speedup=t_dense / t_net if t_net else 1.0)


def replay(controller: GslController, trajectory) -> dict:
    """Drive the controller with rows (iteration, layer, density), checking at every distinct
    iteration in order; returns the report."""
    by_it = {}
    for it, name, x in trajectory:
        by_it.setdefault(int(it), {})[name] = float(x)
    for it in sorted(by_it):
        controller.step(it, {n: x for n, x in by_it[it].items()
                             if controller.layers[n].status == ACTIVE})
    return controller.report()
