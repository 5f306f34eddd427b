"""Global ordering across ranks (oracle c13; test infrastructure only).

BASELINE.json: "one NCCL allgather over NVLink per scheduling round so the
global utility ordering stays exact".  Reading AMB-22: the global order is the
(Pri desc, arrival asc, global id asc) sort over the UNION of all ranks'
waiting sets; the merge of per-rank top-K lists must equal its top-K (the top
K of a union is contained in the union of per-rank top Ks).
"""


def key(rec):
    pri, arrival, rid = rec[0], rec[1], rec[2]
    return (-pri, arrival, rid)


def global_topk(union, K):
    return sorted(union, key=key)[:K]


def merge_rank_topk(per_rank_lists, K):
    allrec = [r for lst in per_rank_lists for r in lst]
    return sorted(allrec, key=key)[:K]
