"""B200-native swept-volume proxy (arXiv 2402.15281 hot path) behind the reference's
inference API.  See DESIGN.md."""
from .program import Layer, LayerProgram, deepsdf, fig2, plain  # noqa: F401
from .api import (Model, MultiModel, QueryResult, batched_proxy, init_params, kernel_timing_begin,  # noqa: F401
                  kernel_timing_end, keys_finalize_device, keys_init_device, launch_count, launch_count_reset, whole_batch)
from .abi import ReferenceInvalidArgument, SvnError  # noqa: F401

__version__ = "0.1.0"
