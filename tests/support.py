"""Shared fixtures, restating the reference's tests/unit/test_support.hpp.

  all_shapes(leaves)      test_support.hpp:37-53 (Catalan enumeration)
  assign_labels(root)     test_support.hpp:58-74 (thresholds 1..I, classes 1..L)
  grid_records(I)         test_support.hpp:87-93 (every tie and every gap)
  depth_chain_tree(d)     test_support.hpp:100-106
  recursive_oracle        eval_serial.cpp:43-75 (conditional descent, <= left)
  fuzz_shape(seed)        acceptance.cpp:120-128
  Appendix A              SURVEY.md golden hashes, computed with the reference
"""
from __future__ import annotations

import copy

import numpy as np

from paper_1111_1373_b200.tree import LinkedNode, make_leaf, make_split


def clone(node: LinkedNode) -> LinkedNode:
    return copy.deepcopy(node)


_SHAPES = {}


def all_shapes(leaves: int):
    if leaves in _SHAPES:
        return [clone(s) for s in _SHAPES[leaves]]
    if leaves == 1:
        shapes = [make_leaf(0)]
    else:
        shapes = []
        for left in range(1, leaves):
            for l in all_shapes(left):
                for r in all_shapes(leaves - left):
                    shapes.append(make_split(0, 0.0, clone(l), clone(r)))
    _SHAPES[leaves] = shapes
    return [clone(s) for s in shapes]


def assign_labels(root: LinkedNode) -> int:
    queue = [root]
    internal = leaf = 0
    head = 0
    while head < len(queue):
        node = queue[head]
        head += 1
        if node.is_leaf():
            leaf += 1
            node.class_val = leaf
        else:
            internal += 1
            node.attribute = 0
            node.threshold = float(internal)
            queue.append(node.left)
            queue.append(node.right)
    return internal


def grid_records(internal: int) -> np.ndarray:
    return np.array([[0.5 + 0.5 * i] for i in range(2 * internal + 1)], dtype=np.float32)


def depth_chain_tree(depth: int) -> LinkedNode:
    tail = make_leaf(depth + 1)
    for level in range(depth - 1, -1, -1):
        tail = make_split(0, 0.5, make_leaf(level + 1), tail)
    return tail


def recursive_oracle(root: LinkedNode, x: np.ndarray) -> np.ndarray:
    """eval_oracle_recursive: conditional descent, value <= threshold goes left."""
    out = np.empty(len(x), dtype=np.uint32)
    for r, rec in enumerate(np.asarray(x, dtype=np.float32)):
        node = root
        while not node.is_leaf():
            node = node.left if rec[node.attribute] <= np.float32(node.threshold) else node.right
        out[r] = node.class_val
    return out


def fuzz_shape(seed: int):
    depth = 1 + seed % 20
    lo = depth + 1
    cap = 1024 if depth >= 10 else (1 << depth)
    hi = min(cap, lo + 19)
    leaves = lo + (seed * 7) % (hi - lo + 1)
    arity = 1 + (seed * 3) % 8
    classes = 2 + seed % 9
    return depth, leaves, arity, classes


def ceil_log2(d: int) -> int:
    steps, reach = 0, 1
    while reach < d:
        reach *= 2
        steps += 1
    return steps


# SURVEY.md Appendix A (tree spec, data spec, tile, tree_fnv, dataset_checksum,
# labels_fnv, first 8 labels, d_mu)
APPENDIX_A = {
    "paper": ((11, 16, 19, 7, 1), (16384, 19, 2), 4, 0x07c58263dd15bc02, 0x33d552cf6075468f,
              0xc90f17638d0c1525, [4, 2, 4, 2, 0, 0, 2, 0], 2.3063),
    "fixture": ((11, 16, 19, 7, 7), (16384, 19, 11), 4, 0x3cc37a3912b7a487, 0xa2a86c49aa26bf0f,
                0x7630db660cbba825, [0, 5, 5, 4, 5, 2, 4, 5], 2.3975),
    "C1": ((10, 1024, 16, 8, 101), (1000000, 16, 102), 1, 0xbc820314fc831ba3, 0x0b4a827f25f4f984,
           0xe52f8e46c62dc8f1, [6, 2, 7, 1, 4, 7, 0, 0], 10.0),
    "C2": ((24, 256, 32, 8, 201), (16000000, 32, 202), 1, 0xd3f4311916fb5aab, 0xc1c3bfe390ef8783,
           0x9e7e87e9cc15c4e0, [7, 4, 3, 5, 5, 4, 5, 3], 4.9845),
    "C3": ((12, 2048, 8, 8, 301), (2073600, 8, 302), 1, 0x8061f80a6ef36aaa, 0xebf422773585ae31,
           0xd57c3eb045278e36, [3, 7, 7, 2, 5, 3, 3, 4], 10.2054),
    "C4t0": ((12, 1024, 64, 8, 401), (8000000, 64, 499), 1, 0x1e22d39cf9ae4df0, 0xa41565fcae97792f,
             0xec47676079b82da6, [4, 3, 5, 6, 2, 6, 0, 7], 8.0930),
    "C5d8": ((8, 256, 16, 8, 508), (15625000, 16, 5000), 1, 0xdc5da3187c1e1003, 0x5143fdb2e3771b61,
             0xa41b18f5886a3516, [4, 4, 5, 2, 3, 0, 3, 6], 8.0),
    "C5d12": ((12, 4096, 16, 8, 512), (15625000, 16, 5000), 1, 0xf4230c4b89e0eac9, 0x5143fdb2e3771b61,
              0x8a36c71851f61114, [4, 6, 1, 7, 3, 1, 4, 2], 12.0),
    "C5d16": ((16, 4096, 16, 8, 516), (15625000, 16, 5000), 1, 0x9c1769a8f519ba65, 0x5143fdb2e3771b61,
              0x4bbe70e47d70a501, [5, 4, 6, 6, 1, 4, 7, 0], 7.7637),
    "C5d20": ((20, 4096, 16, 8, 520), (15625000, 16, 5000), 1, 0xca261bc67cd84dd1, 0x5143fdb2e3771b61,
              0x894ffd1cd01ac0a5, [3, 0, 0, 5, 0, 2, 3, 5], 7.3201),
}
# C4 forest: trees (12, 1024, 64, 8, 401 + t) for t in 0..127 on data(8e6, 64, 499)
C4_FOREST_CHAIN = 0x45bca80476404d56
C4_FOREST_LABELS_FNV = 0x1b2543c41e436ce0
C4_FOREST_FIRST8 = [4, 7, 6, 1, 2, 6, 1, 7]


def workload(co, name):
    """Generate the Appendix A workload `name` with the oracle generators."""
    tspec, dspec, tile, *_ = APPENDIX_A[name]
    nodes = co.gen_tree(*tspec)
    x = co.gen_dataset(*dspec)
    if tile > 1:
        x = np.tile(x, (tile, 1))
    return nodes, x
