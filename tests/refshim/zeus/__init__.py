"""Import shim: ``import zeus`` resolves to paper_2603_28770_b200.

Used by scripts/run_reference_tests.sh to run the REFERENCE's own unit tests
(pkg/tests/test_*.py, copied at run time into the git-ignored baseline/) against
this package: every ``zeus.<module>`` the tests import is aliased to the
package module of the same name.  Not imported by the product or the pytest
suite.
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))))))

import paper_2603_28770_b200 as _pkg  # noqa: E402
from paper_2603_28770_b200 import (  # noqa: E402,F401
    autodiff, bench, bfgs, cli, driver, fitting, linesearch, objectives, pso, streams)

for _name in ("autodiff", "bench", "bfgs", "cli", "driver", "fitting", "linesearch",
              "objectives", "pso", "streams"):
    sys.modules[f"zeus.{_name}"] = getattr(_pkg, _name)
sys.modules["zeus"] = _pkg
