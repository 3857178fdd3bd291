"""B200-native rotation voting (arXiv 2506.11547): the C-ABI library librotvote
(hand-written sm_100a CUDA) and its thin Python binding.

    from paper_2506_11547_b200 import RotVote
    rv = RotVote(max_n=10**6)
    res = rv.solve(x, y, eps=0.05)     # x, y: float32 CUDA tensors [N,3]
"""
from .rotvote import (DEFAULT_CHAIN, RV_DEGENERATE, RV_MODE_BOUND, RV_MODE_EXACT,  # noqa: F401
                      RV_MODE_FINAL, RV_MODE_BOUND_TC, RV_MODE_FINAL_TC,
                      RV_RECHECKED, RV_REFINED, Plan, Result, RotVote,
                      RotVoteError, grid_candidates, lib, rot_vote_create, rot_vote_destroy,
                      rot_vote_get_unique_id, shard_range, unpack_mask)
