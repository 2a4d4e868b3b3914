"""Import shim: `import multipole_attn` resolves to this package (paper_2506_13059_b200), so the
reference's own unit tests (copied beside the installed reference into baseline/_ref_tests by
__graft_entry__.build()) run unmodified against the B200 implementation.  Test infrastructure only."""

import sys

import paper_2506_13059_b200 as _pkg
from paper_2506_13059_b200 import attention, clustering, core, pipeline, rope  # noqa: F401
from paper_2506_13059_b200 import *  # noqa: F401,F403

for _name, _mod in {"attention": attention, "clustering": clustering, "core": core, "pipeline": pipeline,
                    "rope": rope}.items():
    sys.modules[f"{__name__}.{_name}"] = _mod

__all__ = _pkg.__all__
