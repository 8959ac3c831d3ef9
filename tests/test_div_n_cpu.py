"""div_n (csrc/frontier.cu): a / n correctly rounded from RN(1/n) and two
FMAs (Markstein).  The device code relies on it for every r_light, r_heavy,
lat and fid it emits, so the identity is checked here with the host's IEEE
division and C99 fma on random and near-midpoint cases."""

import os
import shutil
import subprocess

import pytest

SRC = r"""
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static uint64_t s = 0x9e3779b97f4a7c15ull;
static uint64_t rnd(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
int main(int argc, char** argv) {
  long long N = atoll(argv[1]), bad = 0;
  for (long long i = 0; i < N; ++i) {
    double n = (double)(1 + (rnd() % (1ull << (1 + rnd() % 33)))), rn = 1.0 / n, a;
    if (i & 1) {                     /* quotient next to a rounding boundary */
      double q = ldexp((double)((rnd() >> 11) | 1ull << 52), -52 + (int)(rnd() % 60) - 30);
      a = q * n;
      uint64_t b; memcpy(&b, &a, 8); b += (int64_t)(rnd() % 9) - 4; memcpy(&a, &b, 8);
    } else {                         /* counts and numerators of the path */
      a = (i & 2) ? (double)(rnd() % (uint64_t)(n + 1)) : (double)(rnd() >> 11) * 0x1p-53 * n * 64;
    }
    double q0 = a * rn, r = fma(-q0, n, a), q1 = fma(r, rn, q0);
    if (q1 != a / n) ++bad;
  }
  printf("%lld\n", bad);
  return 0;
}
"""


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_div_n_is_correctly_rounded(tmp_path):
    c, exe = tmp_path / "div_n.c", tmp_path / "div_n"
    c.write_text(SRC)
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe), str(c), "-lm"], check=True)
    out = subprocess.run([str(exe), "20000000"], capture_output=True, text=True, check=True)
    assert out.stdout.strip() == "0"
