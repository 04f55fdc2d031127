"""B200-native 4-direction 5x5 Sobel (arXiv 2305.00515) behind the reference's
run_stream interface.  See DESIGN.md and INTEGRATION.md."""
from .api import (  # noqa: F401
    Context, DimMismatch, Error, FilterParams, ImageTooSmall, LaneTooNarrow, NonIntegralWeight,
    NonPositiveParam, ParamOverflow, ParityViolation, Prefetch, StreamResult, Strip, StripPlan,
    alloc_input, alloc_planes, launch, launch_band, launch_batch, launch_count,
    make_stream_taps, materialize, plan_counters, plan_strips, run_stream,
    synth_random_device, validate_params)
from ._abi import Diag, Planes, Taps  # noqa: F401
