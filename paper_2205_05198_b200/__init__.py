"""B200-native sequence-parallel transformer layer with selective recomputation
(arXiv 2205.05198 hot path). The compute lives in libspl.so (sm_100a CUDA + NCCL) behind the
C ABI of include/spl.h; this package is the Python mirror of the reference's seqpar API."""
from ._lib import lib, header_symbols, SplError, SplStateError  # noqa: F401
from .seqpar import (BlockConfig, SeqparLayer, SeqparForward, SeqparBackward,  # noqa: F401
                     seqpar_block_forward, seqpar_block_backward, per_layer_bytes,
                     per_layer_bytes_exact, param_count, PARAM_NAMES, SeqparStack,
                     layer_component_breakdown, percent_of_baseline, total_first_stage_bytes,
                     layer_comm_bytes, seqpar_block_forward_sharded, RankShardedTensor,
                     ReferenceForward, BlockGrads, reference_block_forward,
                     reference_block_backward, attention_interior, all_gather, reduce_scatter,
                     all_reduce, RecomputeStrategy)
from .window import (ModelShape, InfeasibleBudget, in_flight, microbatch_bytes,  # noqa: F401
                     window_plan, stage_timeline, SeqparWindow)
