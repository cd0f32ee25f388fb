"""Particle-swarm phase (pso.py of the reference) on the device.

``init_swarm`` / ``update_swarm`` keep the reference signatures and return
host numpy state (the reference's ``SwarmState``); each call runs the sm_100a
kernels of csrc/pso.cu.  ``zeus_run`` keeps the swarm resident in HBM instead
(engine.SwarmShard) and never round-trips it through the host.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import torch

from . import _device, engine
from .objectives import objective_id
from .streams import ParticleStreams

__all__ = ["PsoParams", "SwarmState", "init_swarm", "update_swarm"]


@dataclass(frozen=True)
class PsoParams:
    """Velocity-update coefficients and sweep count (pso.py:24-44)."""

    w: float = 0.5
    c1_pso: float = 1.2
    c2_pso: float = 1.5
    iter_pso: int = 0

    def __post_init__(self):
        if self.w < 0.0 or self.c1_pso < 0.0 or self.c2_pso < 0.0:
            raise ValueError("PSO coefficients must be non-negative")
        if self.iter_pso < 0:
            raise ValueError("iter_pso must be non-negative")


@dataclass
class SwarmState:
    """Positions, velocities and bests for N particles (pso.py:47-70)."""

    positions: np.ndarray
    velocities: np.ndarray
    personal_best_pos: np.ndarray
    personal_best_val: np.ndarray
    global_best_pos: np.ndarray
    global_best_val: float

    @property
    def n(self) -> int:
        return self.positions.shape[0]

    @property
    def dim(self) -> int:
        return self.positions.shape[1]


def _require_streams(rng) -> ParticleStreams:
    if not isinstance(rng, ParticleStreams):
        raise TypeError("the device swarm regenerates draws from (seed, particle, counter); "
                        "pass streams from make_start_streams")
    return rng


def _to_state(shard: engine.SwarmShard) -> SwarmState:
    return SwarmState(
        positions=_device.from_soa(shard.x),
        velocities=_device.from_soa(shard.v),
        personal_best_pos=_device.from_soa(shard.p),
        personal_best_val=shard.pval.cpu().numpy(),
        global_best_pos=shard.gX.cpu().numpy(),
        global_best_val=float(shard.gbest[0].item()),
    )


def init_swarm(
    f: Callable[[Sequence[float]], float],
    n: int,
    search_range: tuple[float, float],
    rng: ParticleStreams,
    dim: int | None = None,
) -> SwarmState:
    """Uniformly seeded swarm over the search box (pso.py:79-120)."""
    if n < 1:
        raise ValueError("swarm needs at least one particle")
    lower, upper = search_range
    if not lower < upper:
        raise ValueError("search range requires lower < upper")
    rng = _require_streams(rng)
    if dim is None:
        dim = rng.dim
    if rng.uniform_offset() != 0:
        raise ValueError("init_swarm needs fresh streams")
    obj = objective_id(f, dim)
    dev = _device.require_device()
    shard = engine.SwarmShard(obj, dim, n, 0, rng.seed, dev)
    shard.init(lower, upper)
    engine.local_barrier(shard)
    rng.advance_all(2 * dim)
    return _to_state(shard)


def update_swarm(
    state: SwarmState,
    f: Callable[[Sequence[float]], float],
    params: PsoParams,
    rng: ParticleStreams,
) -> SwarmState:
    """One velocity/position sweep over all particles, in place (pso.py:123-164)."""
    rng = _require_streams(rng)
    n, dim = state.n, state.dim
    obj = objective_id(f, dim)
    off = rng.uniform_offset()
    if off % (2 * dim):  # (offset 0: a swarm not made by init_swarm, fresh streams)
        raise ValueError("stream offset does not sit on a sweep boundary")
    sweep = off // (2 * dim) - 1
    dev = _device.require_device()
    shard = engine.SwarmShard(obj, dim, n, 0, rng.seed, dev)
    shard.x.copy_(_device.to_soa(state.positions, dev))
    shard.v.copy_(_device.to_soa(state.velocities, dev))
    shard.p.copy_(_device.to_soa(state.personal_best_pos, dev))
    shard.pval.copy_(torch.from_numpy(np.asarray(state.personal_best_val, dtype=np.float64)))
    shard.gX.copy_(torch.from_numpy(np.asarray(state.global_best_pos, dtype=np.float64)))
    shard.sweeps_done = sweep
    shard.sweep(params.w, params.c1_pso, params.c2_pso)
    engine.local_barrier(shard)
    rng.advance_all(2 * dim)
    new = _to_state(shard)
    state.positions[...] = new.positions
    state.velocities[...] = new.velocities
    state.personal_best_pos[...] = new.personal_best_pos
    state.personal_best_val[...] = new.personal_best_val
    state.global_best_pos = new.global_best_pos
    state.global_best_val = new.global_best_val
    return state
