"""The library's constant-time Morton index map (csrc/qtt_internal.h
morton_natural, used by the fused grid apply) against the bit-by-bit
definition (R18: QTT bit dim*l + a = bit l of coordinate a, x
fastest), on the host: compiled with g++ (no GPU), every dim and level count
up to d = 30, sampled indices."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SRC = r"""
#include "paper_1511_06029_b200/csrc/qtt_internal.h"
#include <cstdio>
int main() {
  long long checked = 0;
  for (int dim = 1; dim <= 3; ++dim)
    for (int lv = 1; dim * lv <= 30; ++lv) {
      const long long N = 1LL << (dim * lv);
      const long long step = N > 200000 ? N / 199999 : 1;
      for (long long q = 0; q < N; q += step) {
        long long c[3] = {0, 0, 0};
        for (int l = 0; l < lv; ++l)
          for (int a = 0; a < dim; ++a) c[a] |= ((q >> (dim * l + a)) & 1) << l;
        long long off = 0;
        for (int a = dim - 1; a >= 0; --a) off = (off << lv) | c[a];
        if (off != qtt::morton_natural(q, dim, lv)) { std::printf("FAIL %d %d %lld\n", dim, lv, q); return 1; }
        ++checked;
      }
    }
  std::printf("ok %lld\n", checked);
  return 0;
}
"""


def test_morton_natural_matches_bit_definition(tmp_path):
    src = tmp_path / "m.cpp"
    src.write_text(SRC)
    exe = tmp_path / "m"
    cuda_inc = "/usr/local/cuda/include"
    r = subprocess.run(["g++", "-std=c++17", "-O1", f"-I{ROOT}", f"-I{cuda_inc}", str(src), "-o", str(exe)],
                       capture_output=True, text=True)
    if r.returncode != 0:
        pytest.fail(r.stderr[-2000:])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
