"""Z/lZ host types: the prime modulus object and the residue formats that
cross the plugin boundary.

Mirrors the reference's public surface for this path:
  * `PrimeModulus` (sldlag/modring.py:44-130): canonical residues in [0, l),
    l an odd probable prime of 2..1024 bits, `check`, `random_residues`,
    fixed little-endian serialization.
  * digit planes (sldlag/vecops.py:22-60): an (N, P) uint64 array, one
    little-endian 16-bit digit per cell, P = ceil(bits(l)/16).
  * 32-bit limbs (N, L) uint32 -- the device's native residue format
    (L = ceil(bits(l)/32)); planes and limbs repack two digits per limb.
"""
import random

import numpy as np

TAG_PLUS_ONE = 0
TAG_MINUS_ONE = 1
TAG_SMALL = 2
TAG_FULL = 3

DIGIT_BITS = 16
DIGIT_MASK = (1 << DIGIT_BITS) - 1

_SMALL_PRIMES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71)


def is_probable_prime(n: int, rounds: int = 40) -> bool:
    """Miller-Rabin with `rounds` bases (error <= 4^-rounds); deterministic
    in n so repeated checks agree."""
    n = int(n)
    if n < 2:
        return False
    for p in _SMALL_PRIMES:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while not d & 1:
        d >>= 1
        s += 1
    rng = random.Random(n ^ 0x5D1A6)
    bases = list(_SMALL_PRIMES[:12])
    bases += [rng.randrange(2, n - 1) for _ in range(max(0, rounds - len(bases)))]
    for a in bases:
        a %= n
        if a < 2:
            continue
        x = pow(a, d, n)
        if x == 1 or x == n - 1:
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def next_prime(n: int) -> int:
    n = int(n) + 1
    while not is_probable_prime(n):
        n += 1
    return n


def prev_prime(n: int) -> int:
    n = int(n) - 1
    while n >= 2 and not is_probable_prime(n):
        n -= 1
    if n < 2:
        raise ValueError("no prime below 2")
    return n


class PrimeModulus:
    """The prime l defining Z/lZ (sldlag/modring.py:44-130)."""

    def __init__(self, ell: int):
        ell = int(ell)
        if ell < 3 or ell % 2 == 0:
            raise ValueError(f"modulus must be an odd prime >= 3, got {ell}")
        if not 2 <= ell.bit_length() <= 1024:
            raise ValueError(f"modulus bit length {ell.bit_length()} outside [2, 1024]")
        if not is_probable_prime(ell, 40):
            raise ValueError(f"{ell} failed the probabilistic primality test")
        self.ell = ell
        self.bit_length = ell.bit_length()
        self.byte_width = (self.bit_length + 7) // 8

    @property
    def limbs(self) -> int:
        return max(1, (self.bit_length + 31) // 32)

    @property
    def digits(self) -> int:
        return digit_count(self.ell)

    def __eq__(self, other):
        return hasattr(other, "ell") and int(other.ell) == self.ell

    def __hash__(self):
        return hash(self.ell)

    def __repr__(self):
        return f"PrimeModulus({self.ell}, bits={self.bit_length})"

    def check(self, a: int) -> int:
        if not 0 <= a < self.ell:
            raise ValueError(f"{a} is not a canonical residue mod {self.ell}")
        return a

    def random_residues(self, rng: np.random.Generator, count: int) -> list:
        """`count` uniform residues, same draw as sldlag/modring.py:98-108:
        (ceil(bits/64)+1) uint64 words per value, most significant last."""
        words = (self.bit_length + 63) // 64 + 1
        raw = rng.integers(0, 2**64, size=(count, words), dtype=np.uint64)
        out = []
        for row in raw.tolist():
            x = 0
            for w in reversed(row):
                x = (x << 64) | w
            out.append(x % self.ell)
        return out

    def residue_to_bytes(self, a: int) -> bytes:
        return int(a).to_bytes(self.byte_width, "little")

    def vector_to_bytes(self, vec) -> bytes:
        w = self.byte_width
        return b"".join(int(a).to_bytes(w, "little") for a in vec)

    def vector_from_bytes(self, data: bytes, count: int) -> list:
        w = self.byte_width
        if len(data) != count * w:
            raise ValueError(f"expected {count * w} bytes, got {len(data)}")
        return [self.check(int.from_bytes(data[i * w:(i + 1) * w], "little")) for i in range(count)]


def as_modulus(mod) -> PrimeModulus:
    """Accept our PrimeModulus, the reference's, or a plain int."""
    if isinstance(mod, PrimeModulus):
        return mod
    if hasattr(mod, "ell"):
        m = PrimeModulus.__new__(PrimeModulus)
        m.ell = int(mod.ell)
        m.bit_length = m.ell.bit_length()
        m.byte_width = (m.bit_length + 7) // 8
        return m
    return PrimeModulus(int(mod))


# -- digit planes (sldlag/vecops.py:22-60) ---------------------------------


def digit_count(x: int) -> int:
    return max(1, (int(x).bit_length() + DIGIT_BITS - 1) // DIGIT_BITS)


def ints_to_planes(values, width: int) -> np.ndarray:
    """Canonical residues -> (N, width) uint64 digit planes."""
    values = list(values)
    n = len(values)
    if not n:
        return np.zeros((0, width), dtype=np.uint64)
    blob = b"".join(int(v).to_bytes(2 * width, "little") for v in values)
    return np.frombuffer(blob, dtype="<u2").reshape(n, width).astype(np.uint64)


def planes_to_ints(planes: np.ndarray) -> list:
    p16 = np.ascontiguousarray(planes, dtype="<u2")
    nb = 2 * p16.shape[1]
    blob = p16.tobytes()
    return [int.from_bytes(blob[i * nb:(i + 1) * nb], "little") for i in range(p16.shape[0])]


def planes_to_bytes(planes: np.ndarray, byte_width: int) -> bytes:
    a8 = np.ascontiguousarray(planes, dtype="<u2").view(np.uint8).reshape(planes.shape[0], -1)
    return a8[:, :byte_width].tobytes()


def bytes_to_planes(data: bytes, count: int, byte_width: int, width: int) -> np.ndarray:
    a8 = np.frombuffer(data, dtype=np.uint8).reshape(count, byte_width)
    pad = np.zeros((count, 2 * width), dtype=np.uint8)
    pad[:, :byte_width] = a8
    return pad.view("<u2").astype(np.uint64)


# -- 32-bit limbs (device format) -------------------------------------------


def ints_to_limbs(values, L: int) -> np.ndarray:
    values = list(values)
    if not values:
        return np.zeros((0, L), dtype=np.uint32)
    blob = b"".join(int(v).to_bytes(4 * L, "little") for v in values)
    return np.frombuffer(blob, dtype="<u4").reshape(len(values), L).copy()


def limbs_to_ints(limbs: np.ndarray) -> list:
    a = np.ascontiguousarray(limbs, dtype="<u4")
    nb = 4 * a.shape[-1]
    blob = a.reshape(-1, a.shape[-1]).tobytes()
    return [int.from_bytes(blob[i * nb:(i + 1) * nb], "little") for i in range(len(blob) // nb)]


def planes_to_limbs(planes: np.ndarray, L: int) -> np.ndarray:
    """(N, P) digit planes -> (N, L) limbs (host-side repack)."""
    p = np.asarray(planes, dtype=np.uint64)
    n, P = p.shape
    d = np.zeros((n, 2 * L), dtype=np.uint32)
    k = min(P, 2 * L)
    d[:, :k] = (p[:, :k] & DIGIT_MASK).astype(np.uint32)
    return d[:, 0::2] | (d[:, 1::2] << 16)


def limbs_to_planes(limbs: np.ndarray, P: int) -> np.ndarray:
    a = np.asarray(limbs, dtype=np.uint32)
    n, L = a.shape
    out = np.zeros((n, max(P, 2 * L)), dtype=np.uint64)
    out[:, 0:2 * L:2] = a & DIGIT_MASK
    out[:, 1:2 * L:2] = a >> 16
    return np.ascontiguousarray(out[:, :P])
