"""TEST INFRASTRUCTURE ONLY -- never imported by the product package.

Stand-in for the three `gmpy2` calls the reference package makes
(`is_prime`, `prev_prime`, `next_prime`; /root/reference/pkg/src/sldlag/
modring.py:59,195 and cli.py:209).  gmpy2 is not installed in this image and
there is no network, so this pure-Python Miller-Rabin lets
`tests/golden/make_golden.py` import the reference to produce golden vectors.
Primality only -- none of these calls is on the SpMV arithmetic path
(SURVEY.md section 8 row c1).
"""
import random

_SMALL = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71]


def is_prime(n, reps=25):
    n = int(n)
    if n < 2:
        return False
    for p in _SMALL:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    rng = random.Random(n)
    bases = _SMALL[:12] + [rng.randrange(2, n - 1) for _ in range(max(0, reps - 12))]
    for a in bases:
        a %= n
        if a < 2:
            continue
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def prev_prime(n):
    n = int(n) - 1
    while not is_prime(n):
        n -= 1
    return n


def next_prime(n):
    n = int(n) + 1
    while not is_prime(n):
        n += 1
    return n


def version():
    return "shim"
