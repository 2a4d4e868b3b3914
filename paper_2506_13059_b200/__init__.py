"""B200-native Multipole Attention decode path, a drop-in for the reference package
`multipole_attn` (/root/reference/pkg/src/multipole_attn/__init__.py:11-34 exports the same names).

    import paper_2506_13059_b200 as multipole_attn
    state = multipole_attn.prefill(trace, cfg)          # GPU blockwise clustering
    out, report = multipole_attn.step(state, q, k, v)   # one decode step on the B200 kernels

The device kernels live in libmpattn.so (C ABI: include/mpattn.h); there is no CPU fallback.
"""

from .core import (
    ConfigError,
    EngineConfig,
    HeadLayout,
    HierarchyConfig,
    KvTrace,
    gen_synthetic,
    load_trace,
    write_trace,
)
from .pipeline import MODES, DecodeReport, EngineState, prefill, run, step

__all__ = [
    "ConfigError",
    "DecodeReport",
    "EngineConfig",
    "EngineState",
    "HeadLayout",
    "HierarchyConfig",
    "KvTrace",
    "MODES",
    "gen_synthetic",
    "load_trace",
    "prefill",
    "run",
    "step",
    "write_trace",
]
