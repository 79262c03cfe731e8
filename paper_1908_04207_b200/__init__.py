"""eagercoll on B200: partial collectives (solo / majority allreduce) and eager-SGD.

A from-scratch sm_100a implementation of the hot path of arXiv 1908.04207's
reference package `eagercoll`, behind the same Python API.  See DESIGN.md.

    from paper_1908_04207_b200 import (CollectiveConfig, AllreduceHandle,
                                       EmulatedWorld, ProcessWorld, train_step)
"""

__version__ = "0.1.0"

import os as _os
import warnings as _warnings

# The persistent engine is resident while other kernels launch.  Under CUDA's
# lazy module loading a kernel's first launch loads its code and waits for the
# device's running kernels -- i.e. forever.  Load eagerly (must precede CUDA
# initialisation; bench.py and the tests set it before importing torch).
if _os.environ.get("CUDA_MODULE_LOADING") != "EAGER":
    import torch as _torch
    if _torch.cuda.is_initialized():
        _warnings.warn("CUDA was initialised with lazy module loading; a kernel first "
                       "launched while an engine runs will block. Set "
                       "CUDA_MODULE_LOADING=EAGER before initialising CUDA.", RuntimeWarning)
    _os.environ["CUDA_MODULE_LOADING"] = "EAGER"

from .collectives import (  # noqa: E402,F401
    FLAVORS, MAJORITY, SOLO, SYNC, AllreduceHandle, CollectiveConfig, CollectiveResult,
    allreduce_majority, allreduce_solo, allreduce_sync, ceil_log2, drive, floor_pow2,
    initiator_for_round, run_allreduce, tree_order_sum,
)
from .eagersgd import (  # noqa: E402,F401
    DivergenceError, GradientBuffer, TrainState, attach_delivery_tracking, finish_step,
    load_state, resync_models, resync_step, save_state, staleness_guard, train_step,
    train_step_async, training_process,
)
from .trace import TraceRecorder  # noqa: E402,F401
from .transport import DelayModel, Sleep, delayed_ranks, inject_delay  # noqa: E402,F401
from .world import EmulatedWorld, ProcessWorld  # noqa: E402,F401
