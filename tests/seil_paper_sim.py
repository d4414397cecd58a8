"""Paper-literal SEIL (Alg. 4 SeilInsert, Alg. 5 SeilSearch) on tiny inputs.

Test helper only: an independent, literal transcription of the paper's list
layout (32-item shared blocks stored once in list i, reference entries in
list j, remainder items duplicated into both lists' misc area with the other
list's ID embedded) and its search. It is used to
pin the oracle's candidate universe U(q) and the DCO identities
(O12): Alg. 5 visited in ascending list order must reach exactly U(q), each id
once, and its scan count must equal DCO_paperSEIL.
"""
from collections import defaultdict

BLK_SZ = 32


def seil_insert(l1, l2):
    """Alg. 4 for one batch: returns {list: {"refs", "shared", "misc"}}."""
    assigns = sorted((int(a), int(b), i) for i, (a, b) in enumerate(zip(l1, l2)))  # line 8
    lists = defaultdict(lambda: {"refs": [], "shared": [], "misc": []})
    i = 0
    while i < len(assigns):
        cell = assigns[i][:2]
        j = i
        while j < len(assigns) and assigns[j][:2] == cell:
            j += 1
        items = [a[2] for a in assigns[i:j]]
        nitems = j - i
        nblocks, nmisc = nitems // BLK_SZ, nitems % BLK_SZ
        li, lj = cell
        bptr = len(lists[li]["shared"])
        for b in range(nblocks):
            lists[li]["shared"].append(items[b * BLK_SZ:(b + 1) * BLK_SZ])
        misc = items[nblocks * BLK_SZ:]
        # embed the other list id (self for single-assigned cells, reading R12)
        lists[li]["misc"].extend((x, lj) for x in misc)
        if li != lj:
            lists[lj]["refs"].append((li, nblocks, bptr))
            lists[lj]["misc"].extend((x, li) for x in misc)
        i = j
    return lists


def seil_search(lists, selected_lists):
    """Alg. 5 in the given visit order: returns (ids kept, DCO scanned)."""
    visited = set()
    kept, dco = [], 0
    for lid in selected_lists:
        lst = lists[lid]
        for other, nblocks, bptr in lst["refs"]:               # lines 6-10
            if other not in visited:
                for b in range(nblocks):
                    blk = lists[other]["shared"][bptr + b]
                    dco += len(blk)
                    kept.extend(blk)
        for blk in lst["shared"]:                               # lines 11-13
            dco += len(blk)
            kept.extend(blk)
        for x, other in lst["misc"]:                            # lines 14-17
            dco += 1
            if other not in visited:                            # RemoveVectorIfVisited
                kept.append(x)
        visited.add(lid)                                        # line 18
    return kept, dco
