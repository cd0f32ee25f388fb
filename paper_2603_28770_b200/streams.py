"""Counter-based per-particle streams (streams.py of the reference).

Particle i's stream is numpy's ``Philox(key=[seed mod 2**64, i])`` consumed in
order; here it is produced on the device by a bit-exact Philox4x64-10
(csrc/zeus_common.cuh): u64 draw k of particle i is word k % 4 of the block
generated from counter (k // 4 + 1, 0, 0, 0).  Nothing is stored per particle
but a draw offset, so the PSO kernels regenerate draws from (seed, i, k).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _capi, _device

__all__ = ["ParticleStreams", "make_start_streams"]

_MASK64 = (1 << 64) - 1


class ParticleStreams:
    """Lazy family of per-particle uniform streams (streams.py:21-45)."""

    def __init__(self, seed: int, n: int, dim: int):
        if n < 1:
            raise ValueError("need at least one particle stream")
        self.seed = int(seed) & _MASK64
        self.n = n
        self.dim = dim
        self._offset = np.zeros(n, dtype=np.int64)  # draws consumed per particle

    def offset(self, i: int) -> int:
        return int(self._offset[i])

    def uniform_offset(self) -> int:
        """The common draw offset of all particles (PSO consumes in lockstep)."""
        off = int(self._offset[0])
        if not np.all(self._offset == off):
            raise ValueError("particle streams are at different positions; the swarm "
                             "kernels need all particles at the same draw offset")
        return off

    def advance_all(self, count: int) -> None:
        self._offset += count

    def generator(self, i: int) -> np.random.Generator:
        """Particle i's stream as a numpy Generator (streams.py:32-39):
        ``Generator(Philox(key=[seed, i]))`` positioned at this family's
        current draw offset for particle i.  The kernels regenerate draws
        from (seed, i, k) on the device, so this is a host VIEW of the same
        stream: draws taken from it do not advance the family's offset (the
        reference's object is the stream itself)."""
        if not 0 <= i < self.n:
            raise IndexError(i)
        key = np.array([self.seed, i], dtype=np.uint64)
        bitgen = np.random.Philox(key=key)
        off = int(self._offset[i])
        bitgen.advance(off // 4)         # whole 4-word blocks
        if off % 4:
            bitgen.random_raw(off % 4)   # into the block
        return np.random.Generator(bitgen)

    def draw_uniform(self, i: int, low: float, high: float, size: int) -> np.ndarray:
        """Next ``size`` uniforms in [low, high) from particle i's stream."""
        if not 0 <= i < self.n:
            raise IndexError(i)
        dev = _device.require_device()
        out = torch.empty(max(size, 1), dtype=torch.float64, device=dev)
        _capi.check(_capi.lib().zeus_philox_uniform(self.seed, i, 1, int(self._offset[i]), size,
                                                    float(low), float(high), out.data_ptr(),
                                                    _device.stream_ptr(dev)), "draw_uniform")
        self._offset[i] += size
        return out[:size].cpu().numpy()


def make_start_streams(seed: int, n: int, dim: int) -> ParticleStreams:
    """Independent reproducible substreams for ``n`` particles (streams.py:48-54)."""
    return ParticleStreams(seed, n, dim)
