"""pytest plugin (measurement only): zero the DiT tolerance constants of the GPU test modules so
every tolerance assertion fails and reports its measured error (for sizing the bounds):
    python -m pytest tests/... -m gpu -p tools.tol_probe_plugin --tb=line -q"""


def pytest_collection_modifyitems(session, config, items):
    for it in items:
        for name in ("EPS_TOL_MAX", "EPS_TOL_MEAN", "TRAJ_TOL"):
            if hasattr(it.module, name):
                setattr(it.module, name, 1e-12)
