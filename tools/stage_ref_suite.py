#!/usr/bin/env python
"""Stage the reference's own hot-path tests, unmodified, for tests/ref_suite/.

    python tools/stage_ref_suite.py          # copy into tests/ref_suite/_staged/
    python tools/stage_ref_suite.py --clean  # remove the staged copy

The copies are git-ignored (reference sources stay out of the history) and travel
to the GPU box inside the gpurun snapshot (file names get a ``ref_`` prefix); tests/ref_suite/conftest.py aliases
``flowpipe`` to this package.  The reference's conftest.py is staged as
ref_conftest.py (its fixtures are re-exported by our conftest).
"""

import os
import shutil
import sys

SRC = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = os.path.join(ROOT, "tests", "ref_suite", "_staged")
MODULES = ["test_velocity.py", "test_schedule.py", "test_pipeline.py", "test_models.py", "test_engine.py"]


def main():
    if "--clean" in sys.argv:
        shutil.rmtree(DST, ignore_errors=True)
        return 0
    os.makedirs(DST, exist_ok=True)
    for m in MODULES:
        # renamed test_x.py -> test_ref_x.py (contents unmodified): pytest's rootdir-relative
        # module names would otherwise clash with tests/test_engine.py
        shutil.copyfile(os.path.join(SRC, m), os.path.join(DST, m.replace("test_", "test_ref_", 1)))
    shutil.copyfile(os.path.join(SRC, "conftest.py"), os.path.join(DST, "ref_conftest.py"))
    print(f"staged {len(MODULES)} reference test modules into {DST}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
