"""Run the reference's OWN hot-path test modules against this package.

``tools/stage_ref_suite.py`` copies /root/reference/pkg/tests/{conftest,test_velocity,
test_schedule,test_pipeline,test_models,test_engine}.py unmodified into
``tests/ref_suite/_staged/`` (git-ignored: reference sources never enter the history;
the staged copy travels to the GPU box with the snapshot).  This conftest makes
``import flowpipe`` resolve to ``paper_2511_22009_b200`` -- the one-line import swap of
INTEGRATION.md section 1 -- loads the reference conftest's fixtures, and marks every
collected test ``gpu`` (the package computes only through libstreamflow.so on a
CUDA device).  Without a staged copy nothing is collected.
"""

import importlib.util
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
STAGED = os.path.join(HERE, "_staged")

import paper_2511_22009_b200 as _pkg  # noqa: E402

sys.modules["flowpipe"] = _pkg
for _sub in ("errors", "schedule", "velocity", "models", "pipeline", "engine"):
    sys.modules["flowpipe." + _sub] = getattr(_pkg, _sub)

_ref_conftest = os.path.join(STAGED, "ref_conftest.py")
if os.path.exists(_ref_conftest):
    spec = importlib.util.spec_from_file_location("flowpipe_ref_conftest", _ref_conftest)
    _mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(_mod)
    for _name in dir(_mod):
        _obj = getattr(_mod, _name)
        if hasattr(_obj, "_pytestfixturefunction") or type(_obj).__name__ == "FixtureFunctionDefinition":
            globals()[_name] = _obj


def pytest_ignore_collect(collection_path, config):
    p = str(collection_path)
    return p.endswith(".py") and os.path.basename(p).startswith("test_") and os.sep + "_staged" + os.sep not in p


def pytest_collection_modifyitems(config, items):
    for it in items:
        if os.sep + "ref_suite" + os.sep in str(it.fspath):
            it.add_marker(pytest.mark.gpu)
