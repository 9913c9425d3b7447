"""Counter-based random streams for the device filter.

The reference threads one ``numpy.random.Generator`` through the filter and
consumes it sequentially (init ``normal(0,σ,(N,2))``, per frame
``normal(0,1,(N,5))`` then ``random()`` iff resampling). A sequential host
generator cannot feed a device kernel, so the device path uses Philox4x32-10
keyed by a 64-bit seed, with the counter = (particle index, frame, stream
tag). Draws depend only on (seed, frame, particle), never on launch order or
the number of GPUs.

``as_philox`` accepts either a :class:`PhiloxRng` or a numpy ``Generator``;
a Generator is converted by drawing one 63-bit key from it, so code written
against the reference (``rng = np.random.default_rng(42)``) stays
deterministic under its seed.
"""

from dataclasses import dataclass, field

import numpy as np

from . import _lib

RESAMPLE_STANDALONE_BASE = 1 << 31   # frame ids for resample() outside a track


@dataclass
class PhiloxRng:
    """Counter-based stream handle: ``seed`` plus the next frame index."""

    seed: int
    frame: int = 0
    resample_calls: int = field(default=0)

    def next_frame(self):
        """Frame id for the next propagation (one per sis/pc_sis step)."""
        f = self.frame
        self.frame += 1
        return f

    def resample_u(self, frame=None):
        """Systematic offset u in [0,1) (filtering.py:99 ``rng.random()``)."""
        if frame is None:
            frame = RESAMPLE_STANDALONE_BASE + self.resample_calls
            self.resample_calls += 1
        return float(_lib.lib().pcs_philox_resample_u(self.seed & (2 ** 64 - 1),
                                                      frame & 0xFFFFFFFF))

    def multinomial_frame(self):
        f = RESAMPLE_STANDALONE_BASE + self.resample_calls
        self.resample_calls += 1
        return f


class ReplayNormals:
    """Feeds recorded (N,5) standard normals (e.g. a reference run's
    ``rng.normal(size=(N,5))`` draws) to the next propagations instead of
    Philox draws — the device arithmetic is unchanged (pcs_propagate_given)."""

    def __init__(self, *normals_n5):
        self._queue = [np.asarray(z, dtype=np.float32) for z in normals_n5]

    def replay_normals(self, n):
        z = self._queue.pop(0)
        if z.shape != (n, 5):
            raise ValueError("recorded normals must have shape (N, 5)")
        return np.ascontiguousarray(z.T)


def as_philox(rng):
    if isinstance(rng, PhiloxRng):
        return rng
    if isinstance(rng, np.random.Generator):
        return PhiloxRng(int(rng.integers(0, 2 ** 63 - 1)))
    if isinstance(rng, (int, np.integer)):
        return PhiloxRng(int(rng))
    raise TypeError(f"unsupported rng {type(rng).__name__}; pass a PhiloxRng, int seed "
                    "or numpy Generator")
