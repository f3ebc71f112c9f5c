"""pytest plugin (-p seam_plugin): run the reference package's own tests with
its kernel seam routed to the B200 library -- INTEGRATION.md §2's setattr on
`fieldbridge._kernels` (reference _kernels/__init__.py:9-42), done before any
test module imports `fieldbridge.pointwise` / `locate` (which resolve
`_kernels.<fn>` at call time, pointwise.py:17, 175, 240, 256, 302;
locate.py:182).  Each routed call is counted; FM_SEAM_REPORT names a JSON
file that receives the counts, so the caller can check the GPU path ran."""

import json
import os

NAMES = ("rbf_weights", "fixed_radius_supports", "adaptive_radius_supports", "fit_many",
         "locate_batch")
CALLS = {}


def pytest_configure(config):
    import fieldbridge._kernels as K

    from paper_2510_18838_b200 import _kernels as B

    for name in NAMES:
        fn = getattr(B, name)

        def routed(*args, _fn=fn, _name=name, **kwargs):
            CALLS[_name] = CALLS.get(_name, 0) + 1
            return _fn(*args, **kwargs)

        setattr(K, name, routed)
    K.BACKEND = B.BACKEND


def pytest_unconfigure(config):
    out = os.environ.get("FM_SEAM_REPORT")
    if out:
        with open(out, "w") as f:
            json.dump(CALLS, f)
