"""pytest plugin: run the reference's own test files against the drop-in.

Loaded with ``-p drop_in_alias`` (PYTHONPATH = this directory, the repo root
and baseline/_ref).  It imports the unmodified reference package ``evsim``
from baseline/_ref and then points ``evsim.events`` (and its submodules
``types``, ``model``, ``parallel``) at ``paper_2602_15018_b200.events``, so
every ``from evsim.events import ...`` in the reference's tests, helpers and
callers (SimNode, orchestrator.py:32-42) resolves to the B200 implementation.
The other reference subsystems (rendering, dynamics, messaging) stay the
reference's own.  This is exactly the backend switch INTEGRATION.md
describes, done at import time instead of by editing the reference.
"""

from __future__ import annotations

import sys

import evsim  # the reference package (baseline/_ref)

import paper_2602_15018_b200.events as _ev
from paper_2602_15018_b200.events import model as _model
from paper_2602_15018_b200.events import parallel as _parallel
from paper_2602_15018_b200.events import types as _types

sys.modules["evsim.events"] = _ev
sys.modules["evsim.events.types"] = _types
sys.modules["evsim.events.model"] = _model
sys.modules["evsim.events.parallel"] = _parallel
evsim.events = _ev


def pytest_terminal_summary(terminalreporter):
    import evsim.events as active

    terminalreporter.write_line(f"drop-in active: evsim.events -> {active.__name__} "
                                f"(generate_events_parallel from {active.generate_events_parallel.__module__})")
