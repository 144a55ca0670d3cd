"""TEST INFRASTRUCTURE ONLY — CPU restatement of numpy's PCG64 streams.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module; it is the checker for the GPU sampler's RNG, never the
thing measured or shipped.

The reference (kgdist) draws every sampled index stream from
`numpy.random.default_rng` (PCG64, numpy 2.x):
  - sampler.py:164    `rng.random(n) < 0.5`            (one next64 per element)
  - sampler.py:173    `rng.integers(len(pool), size=k)` (32-bit Lemire on the
                                                         buffered next_uint32)
  - sampler.py:220    `rng.permutation(total)`          (Fisher-Yates, masked
                                                         rejection on next_uint32)
  - model.py:225      `dropout_rng.random(A.shape)`
numpy is an un-vendored dependency (pyproject.toml:10-13 pins only
`numpy>=1.24`); the algorithms restated here are numpy's published
implementation (numpy/random/src/pcg64/pcg64.h and
numpy/random/src/distributions/distributions.c). They are pinned against the
numpy present in this container by tests/test_oracle_rng.py.
"""

from __future__ import annotations

MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


class PCG64Stream:
    """Bit-exact emulation of numpy's PCG64 + Generator draw helpers."""

    def __init__(self, state: int, inc: int, has_uint32: int = 0, uinteger: int = 0):
        self.state = state & MASK128
        self.inc = inc & MASK128
        self.has_uint32 = int(has_uint32)
        self.uinteger = int(uinteger) & 0xFFFFFFFF

    # -- construction from / export to numpy's state dict ------------------
    @classmethod
    def from_numpy(cls, gen) -> "PCG64Stream":
        st = gen.bit_generator.state
        return cls(st["state"]["state"], st["state"]["inc"], st["has_uint32"], st["uinteger"])

    def numpy_state(self) -> dict:
        return {"bit_generator": "PCG64",
                "state": {"state": self.state, "inc": self.inc},
                "has_uint32": self.has_uint32, "uinteger": self.uinteger}

    # -- raw outputs --------------------------------------------------------
    def next64(self) -> int:
        # step first, then XSL-RR output of the new state
        self.state = (self.state * PCG_MULT + self.inc) & MASK128
        s = self.state
        rot = s >> 122
        x = ((s >> 64) ^ s) & MASK64
        return ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64

    def next32(self) -> int:
        if self.has_uint32:
            self.has_uint32 = 0
            return self.uinteger
        v = self.next64()
        self.has_uint32 = 1
        self.uinteger = v >> 32
        return v & 0xFFFFFFFF

    def advance(self, delta: int) -> None:
        """Jump the LCG ahead by `delta` steps (== delta next64 calls)."""
        acc_mult, acc_plus = 1, 0
        cur_mult, cur_plus = PCG_MULT, self.inc
        delta &= MASK128
        while delta:
            if delta & 1:
                acc_mult = (acc_mult * cur_mult) & MASK128
                acc_plus = (acc_plus * cur_mult + cur_plus) & MASK128
            cur_plus = ((cur_mult + 1) * cur_plus) & MASK128
            cur_mult = (cur_mult * cur_mult) & MASK128
            delta >>= 1
        self.state = (acc_mult * self.state + acc_plus) & MASK128

    # -- Generator helpers --------------------------------------------------
    def random(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def lemire32(self, n: int) -> int:
        """integers(n) for 1 < n <= 2**32 - 1 (numpy: buffered_bounded_lemire_uint32)."""
        rng_excl = n
        m = self.next32() * rng_excl
        leftover = m & 0xFFFFFFFF
        if leftover < rng_excl:
            threshold = ((1 << 32) - rng_excl) % rng_excl
            while leftover < threshold:
                m = self.next32() * rng_excl
                leftover = m & 0xFFFFFFFF
        return m >> 32

    def integers(self, n: int, size: int) -> list:
        if n == 1:
            return [0] * size
        return [self.lemire32(n) for _ in range(size)]

    def interval(self, mx: int) -> int:
        """numpy random_interval(max): masked rejection on next_uint32."""
        if mx == 0:
            return 0
        mask = mx
        for sh in (1, 2, 4, 8, 16, 32):
            mask |= mask >> sh
        while True:
            v = self.next32() & mask
            if v <= mx:
                return v

    def permutation_swaps(self, n: int) -> list:
        """The Fisher-Yates swap targets j_i for i = n-1 .. 1 (in that order)."""
        return [self.interval(i) for i in range(n - 1, 0, -1)]

    def permutation(self, n: int) -> list:
        arr = list(range(n))
        for i in range(n - 1, 0, -1):
            j = self.interval(i)
            arr[i], arr[j] = arr[j], arr[i]
        return arr


def lemire_threshold(n: int) -> int:
    return ((1 << 32) - n) % n


def resolve_permutation(js: list, n: int) -> list:
    """Order-free resolution of the Fisher-Yates swap chain (the algorithm the
    GPU kernel implements): given j_i for i=n-1..1, return
    the final permutation of arange(n) without replaying the swaps."""
    jof = {}
    for k, j in enumerate(js):
        jof[n - 1 - k] = j
    groups = {}
    for i in range(n - 1, 0, -1):
        groups.setdefault(jof[i], []).append(i)
    for g in groups.values():
        g.sort()

    def T(p):
        for i in groups.get(p, []):
            if i > p:
                return i
        return None

    def root(p):
        while True:
            t = T(p)
            if t is None:
                return p
            p = t

    out = [0] * n
    out[0] = root(0)
    for i in range(1, n):
        j = jof[i]
        g = groups[j]
        k = g.index(i)
        s = g[k + 1] if k + 1 < len(g) else None
        out[i] = root(s) if s is not None else (root(i) if j == i else j)
    return out
