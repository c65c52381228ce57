"""CPU oracle for the Purine data-parallel hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy float32, the reference algorithm of
every operator kind on the data-parallel SGD path of the reference
(`/root/reference/pkg/src/biflow/ops.py`) plus the kinds the reference lacks
but the GoogLeNet/NIN configurations need (pooling, LRN, concat, momentum
SGD, floor-mode convolution).  It also restates the reference's serial-mode
dispatch order (`dispatcher.py:96-206`).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package, and
only as the checker or the CPU baseline — never as the product path.  The
product package ``paper_1412_6249_b200`` must never import it.

Pinning:
  * reference kinds (fc, conv, relu, flatten, softmax_xent, sgd_update,
    aggregate, copy, swap): pinned against golden vectors produced by the
    reference itself (``tests/golden/make_golden.py`` imports ``biflow`` from
    ``/root/reference`` in the build container) and against the frozen
    scalars of ``pkg/tests/test_ops.py``.
  * extension kinds (maxpool, avgpool, lrn, concat, sgd_momentum,
    floor-mode conv): the reference has no implementation, so these are
    **parity unpinned** by the reference; they are pinned by the golden tiny
    cases, loop oracles and finite differences in ``tests/test_oracle.py``.
"""

from .kernels import *  # noqa: F401,F403
from .kernels import __all__ as _k_all
from .serial import (serial_order, run_graph_lanes, run_graph_serial,  # noqa: F401
                     run_sequence_serial)

__all__ = list(_k_all) + ["serial_order", "run_graph_serial", "run_graph_lanes",
                          "run_sequence_serial"]
