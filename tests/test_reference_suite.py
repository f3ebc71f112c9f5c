"""The reference's own pointwise + locate tests through the B200 seam (-m gpu).

/root/reference/pkg/tests/test_pointwise.py and test_locate.py, with the
reference package (built by `make -C oracle refpkg` into the git-ignored
oracle/_ref/pkg, which travels to the GPU box), run in a subprocess with
tests/seam_plugin.py routing fieldbridge._kernels.{rbf_weights,
fixed_radius_supports, adaptive_radius_supports, fit_many, locate_batch} to
paper_2510_18838_b200._kernels (libfieldmap.so).  Every test must pass, and
every routed name must have been called (the GPU path ran)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

PKG = os.path.join(ROOT, "oracle", "_ref", "pkg")

pytestmark = pytest.mark.gpu


def test_reference_pointwise_and_locate_tests_through_the_seam(tmp_path):
    if not os.path.isdir(os.path.join(PKG, "tests")):
        pytest.fail("oracle/_ref/pkg missing: run `make -C oracle refpkg` (needs /root/reference)")
    report = tmp_path / "seam.json"
    env = dict(os.environ, FM_SEAM_REPORT=str(report),
               PYTHONPATH=os.pathsep.join([PKG, ROOT, os.path.join(ROOT, "tests")]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "seam_plugin", "-p", "no:cacheprovider",
           "--rootdir", PKG, os.path.join(PKG, "tests", "test_pointwise.py"),
           os.path.join(PKG, "tests", "test_locate.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=PKG)
    print(res.stdout[-3000:], res.stderr[-2000:])
    assert res.returncode == 0, res.stdout[-3000:]
    calls = json.loads(report.read_text())
    for name in ("rbf_weights", "fixed_radius_supports", "adaptive_radius_supports",
                 "fit_many", "locate_batch"):
        assert calls.get(name, 0) > 0, calls
    passed = [ln for ln in res.stdout.splitlines() if " passed" in ln]
    assert passed, res.stdout[-500:]
