"""B200-native DET-LSH hot path (arxiv 2603.24920): DE-Tree build + batched c^2-k-ANN.

The CUDA library ``libdetlsh.so`` (C ABI in include/detlsh.h) does all the work; this
package is the thin Python binding (``detlsh``) and the multi-GPU glue (``dist``).
"""
from .detlsh import (DetlshError, Index, MODE_CELL, MODE_EXACT, MODE_RELAXED, STATS_DTYPE, build, default_opts,  # noqa: F401
                     detlsh_breakpoints_from_samples, detlsh_build, detlsh_build_from_codes,
                     detlsh_load, detlsh_merge_topk, detlsh_query_candidates, candidate_ids, detlsh_params, detlsh_query, detlsh_query_ex,
                     detlsh_sample_projections, detlsh_sample_size, launch_count, lib, profile_enable,
                     profile_filter, profile_read, profile_reset, release_workspace, workspace_bytes)
