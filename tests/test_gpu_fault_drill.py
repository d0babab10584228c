"""The suites can fail: with the reference's fault injection
(MOE_FAULT_INJECT=i2f4 / i2f8 shifts the int4 / int8 debias constant by one
code, proj/src/dequant.cpp:12-30 and proj/tests/python/test_cli.py:97-108)
the GPU dequant and both layer modes must disagree with the oracle; without
it they agree (the same probe, un-faulted)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

PROBE = os.path.join(ROOT, "tests", "fault_drill_probe.py")


def _probe(bits, fault):
    env = dict(os.environ)
    env.pop("MOE_FAULT_INJECT", None)
    if fault:
        env["MOE_FAULT_INJECT"] = fault
    r = subprocess.run([sys.executable, PROBE, str(bits)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("bits,fault", [(4, "i2f4"), (8, "i2f8")])
def test_fault_injection_breaks_parity(cuda, bits, fault):
    res = _probe(bits, fault)
    assert res["debias_u4" if bits == 4 else "debias_u8"] == ("0x6409" if bits == 4 else "0x6481")
    assert not res["dequant_equal"], res
    assert not res["exact_equal"], res
    assert res["fast_err"] > 1e-2, res


@pytest.mark.parametrize("bits", [4, 8])
def test_without_fault_parity_holds(cuda, bits):
    res = _probe(bits, None)
    assert res["dequant_equal"] and res["exact_equal"], res
    assert res["fast_err"] <= 1e-2, res
