"""Host-side exhaustive checks behind two device-numerics claims (DESIGN.md
§4), compiled with gcc and run on CPU:

* quant_div_check.c -- the quantizer's f32 division + round-half-away gives
  the reference's llround(f64 w / f64 s) code for EVERY (fp16 w, fp16 s)
  pair that does not clamp (proj/src/quantize.cpp:26-32), int4 and int8;
* expf_check.c -- the device port of glibc expf (csrc/glibc_expf.h) equals
  the host libm expf bit for bit (here over a 2^24-pattern slice of the
  gate's domain, non-positive inputs; the full 2^32 sweep is the same binary
  without arguments)."""
import os
import subprocess

import pytest

from conftest import ROOT

NATIVE = os.path.join(ROOT, "tests", "native")
CSRC = os.path.join(ROOT, "paper_2211_10017_b200", "csrc")


def _build(tmp_path, src, *extra):
    exe = str(tmp_path / os.path.splitext(src)[0])
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-I", CSRC, "-o", exe,
                    os.path.join(NATIVE, src), *extra, "-lm", "-lpthread"], check=True)
    return exe


def test_quantizer_f32_division_exhaustive(tmp_path):
    exe = _build(tmp_path, "quant_div_check.c")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 mismatches" in r.stdout


def test_expf_port_slice(tmp_path):
    exe = _build(tmp_path, "expf_check.c")
    r = subprocess.run([exe, "0xC0800000", "0xC1800000"], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches=0 " in r.stdout, r.stdout
