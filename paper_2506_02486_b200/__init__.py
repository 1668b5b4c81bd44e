"""B200-native DiOMP-Offloading hot path.

Drop-in for the reference package's public surface (reference/pkg/src/diomp/
__init__.py:10-23): init()/finalize(), Runtime (alloc_symmetric /
alloc_asymmetric / free / translate / resolve_cell / put / get / fence /
barrier / groups), the OMPCCL collectives, the kernel seam and the Minimod /
Cannon / bench drivers.  Segments live in B200 HBM, peers are reached over
NVLink, and every data-path operation is a hand-written sm_100a kernel in
libdiomp_b200.so (include/diomp_b200.h).  `import paper_2506_02486_b200 as
diomp` is the intended spelling for reference users.
"""

from . import errors
from .errors import *  # noqa: F401,F403
from .global_memory import (AllocatorKind, AllocMode, AllocRecord, GlobalAddress, GlobalMemory,
                            IndirectionCell, Segment, SegmentConfig, TransferKind,
                            segment_create)
from .config import LaunchConfig, ResolvedConfig, resolve_from_env
from .topology import Endpoint, PathKind, TopologyMap, classify_path
from .streams import Stream, StreamEvent, StreamPool
from .runtime import (CompletionHandle, Group, HandleState, Runtime, StreamedHandle, finalize,
                      init)
from . import collectives, kernels
from .wire import Status
from .collectives import (Communicator, ElementType, ReduceKind, ReduceOp, UniqueId, allreduce,
                          bcast, bootstrap, device_bcast, reduce)

__version__ = "0.1.0"
