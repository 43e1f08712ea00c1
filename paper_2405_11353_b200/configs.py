"""The BASELINE.json workloads (configs[0..4] -> config 1..5) and their
seeded synthetic inputs (uniform residues in [0,P) from
``np.random.default_rng(k)``; the reference measures on synthetic sizes only,
PAPER.md:361, so no dataset is involved)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

P998 = 998244353
GOLD = (1 << 64) - (1 << 32) + 1


@dataclass(frozen=True)
class Workload:
    cfg: int
    seed: int
    batch: int
    log2n: int
    p: int
    g: int
    w: int
    variants: tuple
    inverse_too: bool
    n1: int | None = None

    @property
    def n(self) -> int:
        return 1 << self.log2n

    @property
    def word(self) -> int:
        return 4 if self.p < (1 << 32) else 8

    @property
    def dtype(self):
        return np.uint32 if self.word == 4 else np.uint64

    def algorithmic_bytes(self, directions: int = 1) -> int:
        """2*N*W per transform (one compulsory read + one write), SURVEY sec.8d."""
        return directions * self.batch * 2 * self.n * self.word

    def butterflies(self, directions: int = 1) -> int:
        return directions * self.batch * (self.n // 2) * self.log2n


CONFIGS = {
    1: Workload(1, 1, 1, 10, P998, 3, 32, ("naive", "dit", "dif", "flat", "pease", "pease_nc", "stockham", "sixstep"), True),
    2: Workload(2, 2, 4096, 12, P998, 3, 32, ("dit", "pease_nc"), False),
    3: Workload(3, 3, 256, 16, GOLD, 7, 64, ("dif",), True),
    4: Workload(4, 4, 512, 20, P998, 3, 32, ("pease_nc",), False),
    5: Workload(5, 5, 1, 26, GOLD, 7, 64, ("sixstep",), False, n1=1 << 13),
}

# survey golden hashes (computed by running the reference itself)
GOLDEN = {
    1: ("b9a1048979ae312b06a2bebc7de559b494228fa2465b6ed275ea624e2f918102",
        "0aeed7d1270fec3ea094c12bc02cac5bca549d284b6915b588d4c058fe3a4ef5"),
    2: ("f311ff6020bf6835450407dea19745b07f04a0d8c992b365aa744b9e988e447a",
        "6aa7cdd658fc1c28a06b3da61aa66bf6e479566ba634fb35138049147bf20dd2"),
    3: ("2f0ceaca214ecc1507d16cebabd64a88850bc54ca97c45b3f249781f996c3991",
        "cea44cfc739c4c63aad8d80f13b88b1b6a10f42ce41af47d648d357e71aed485"),
    4: ("949b930a80ac178bf5ae11d39ae51cceb36d2d86cbaaaccc7d0e3a055e5486f3",
        "c66de26c6d584de8144c2a03d5b799c0bac18a3ef0b771b0fdc2c75759bfbc9c"),
    5: ("451e26e5af2f0636823ecf7452db1e4a6e35708d4a63d642b489e090acf13604",
        "039c248452f97c8b5b76ca4c8ca2b7609260a93079335eb81afe8f9fe0c60f4e"),
}


def seeded_input(w: Workload, rows: int | None = None) -> np.ndarray:
    """np.random.default_rng(seed).integers(0, P, size=(B, N), dtype=uint64),
    cast to uint32 for P < 2^32 (shape-independent stream: the first `rows`
    rows equal the first rows of the full draw)."""
    b = w.batch if rows is None else rows
    x = np.random.default_rng(w.seed).integers(0, w.p, size=(b, w.n), dtype=np.uint64)
    return x.astype(np.uint32) if w.word == 4 else x


def seeded_rows(w: Workload, lo: int, hi: int, chunk: int = 1024) -> np.ndarray:
    """Rows [lo, hi) of the seeded stream of ``seeded_input`` -- for a batch of
    any size (the stream is shape-independent), so rank r of a weak-scaling run
    transforms rows [r*B, (r+1)*B) of ONE global seeded batch and rank 0's rows
    are exactly the config's own input.  Rows before `lo` are drawn and
    discarded in chunks (bounded memory)."""
    rng = np.random.default_rng(w.seed)
    skip = lo
    while skip:
        k = min(chunk, skip)
        rng.integers(0, w.p, size=(k, w.n), dtype=np.uint64)
        skip -= k
    x = rng.integers(0, w.p, size=(hi - lo, w.n), dtype=np.uint64)
    return x.astype(np.uint32) if w.word == 4 else x
