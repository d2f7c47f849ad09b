"""The reference's OWN test files, unmodified, run against the drop-in.

tools/install_reference.sh puts the reference package and its test suite in
the git-ignored baseline/_ref (it travels to the GPU box); tests/drop_in_alias.py
aliases ``evsim.events`` to ``paper_2602_15018_b200.events`` before the
reference's tests import it.  Each file runs in its own pytest process from
a copy of the reference's package directory (the tests open
configs/default.yaml and golden/ relative to it).  Skipped when baseline/_ref
has not been installed.
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
PKG = os.path.join(REF, "pkg_tests")

needs_ref = pytest.mark.skipif(not os.path.isdir(os.path.join(PKG, "tests")),
                               reason="reference not installed (tools/install_reference.sh)")


def _env(alias: bool):
    env = dict(os.environ)
    paths = [os.path.join(PKG, "tests"), REF, ROOT]
    if alias:
        paths.insert(0, os.path.join(ROOT, "tests"))
    env["PYTHONPATH"] = os.pathsep.join(paths + [env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    return env


def _pytest(args, alias=True, timeout=900):
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "no:randomly",
           "--rootdir", PKG, "-c", os.devnull]
    if alias:
        cmd += ["-p", "drop_in_alias"]
    r = subprocess.run(cmd + args, cwd=PKG, env=_env(alias), capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout + r.stderr


@needs_ref
@pytest.mark.parametrize("target", [
    "tests/test_event_model.py",
    "tests/test_event_parallel.py",
    # the event-path release criteria (test_acceptance.py:79-150) and the
    # SimNode determinism criterion, through the drop-in
    "tests/test_acceptance.py::test_oracle_equivalence",
    "tests/test_acceptance.py::test_atomic_reduction",
    "tests/test_acceptance.py::test_contrast_model_correctness",
    "tests/test_acceptance.py::test_determinism",
    # SimNode stepping with the drop-in behind it (orchestrator.py:143-177),
    # incl. the serial == parallel backend hash (test_orchestrator.py:110-114)
    "tests/test_orchestrator.py::TestStepOnce",
    "tests/test_orchestrator.py::TestApplyZoh",
])
def test_reference_suite_against_drop_in(target):
    rc, out = _pytest([target, "-p", "no:warnings"])
    assert rc == 0, out[-4000:]
    assert ("drop-in active: evsim.events -> paper_2602_15018_b200.events "
            "(generate_events_parallel from paper_2602_15018_b200.events.parallel)") in out, out[-2000:]
    assert " passed" in out and " failed" not in out, out[-2000:]


_HASH = r"""
import sys
sys.path.insert(0, "tests")
from test_orchestrator import _base_doc, _bundle_hash
from evsim.sim import SimNode, config_from_dict
for backend in ("parallel", "serial"):
    doc = _base_doc(event_backend=backend, seed=7)
    doc["trajectory"] = {"type": "circle", "center": [0, 0, 1.0], "radius": 1.0, "omega": 3.0}
    doc["event_camera"]["sigma_c"] = 0.03
    doc["event_camera"]["noise_rate_hz"] = 50.0
    node = SimNode(config_from_dict(doc))
    n = sum(len(node.step_once().events) for _ in range(5))
    print(backend, n, _bundle_hash(SimNode(config_from_dict(doc)), 20))
"""


@needs_ref
def test_simnode_bundles_identical_to_reference():
    """SimNode (renderer + dynamics + events + noise, orchestrator.py:143-196)
    flying a circle (events every tick, sigma_c 0.03, 50 Hz noise) over 20
    ticks, both event backends: the hash of every published bundle with the
    unmodified reference equals the hash with evsim.events replaced by the
    drop-in (the reference's backend-equality check, test_orchestrator.py:110-114,
    across implementations)."""
    outs = []
    for alias in (False, True):
        pre = "import drop_in_alias\n" if alias else ""
        r = subprocess.run([sys.executable, "-c", pre + _HASH], cwd=PKG, env=_env(alias), capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        outs.append(r.stdout.strip())
    assert outs[0] == outs[1], outs
    lines = outs[0].splitlines()
    assert len(lines) == 2 and all(int(ln.split()[1]) > 0 for ln in lines), outs
