"""Tree model: the reference's tree-load boundary (core/include/spectree/tree.hpp).

``EncodedTree`` holds the breadth-first node array in exactly the reference's
16-byte ``EncodedNode`` layout (tree.hpp:43-55) as a numpy structured array,
so it can be handed to the C ABI without conversion.  Derived stats follow
the reference constructor (tree.cpp:35-61): leaf count, depth in edges,
``max_attribute`` over *all* nodes (leaves included, tree.cpp:47) and the
ascending internal index list (the processor-node map, tree.cpp:204-209).
"""
from __future__ import annotations

import json
import math
import threading
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .errors import ArgumentError, SchemaError, StructureError

NO_CLASS = 0xFFFFFFFF  # kNoClass, tree.hpp:15-16
NODE_DTYPE = np.dtype(
    [("attribute", "<u4"), ("threshold", "<f4"), ("child", "<u4"), ("class_id", "<u4")]
)
assert NODE_DTYPE.itemsize == 16


@dataclass
class LinkedNode:
    """Pointer-linked full binary tree node (tree.hpp:21-29)."""

    attribute: int = 0
    threshold: float = 0.0
    class_val: Optional[int] = None
    left: Optional["LinkedNode"] = None
    right: Optional["LinkedNode"] = None

    def is_leaf(self) -> bool:
        return self.left is None and self.right is None


def make_leaf(class_val: int) -> LinkedNode:  # tree.cpp:11-19
    if class_val == NO_CLASS:
        raise ArgumentError(f"class id {NO_CLASS} is reserved as the no-class sentinel")
    return LinkedNode(class_val=class_val)


def make_split(attribute: int, threshold: float, left: LinkedNode, right: LinkedNode) -> LinkedNode:
    if left is None or right is None:  # tree.cpp:21-33
        raise ArgumentError("split node requires both children")
    return LinkedNode(attribute=attribute, threshold=threshold, left=left, right=right)


class EncodedTree:
    """Breadth-first array encoding (tree.hpp:61-92)."""

    def __init__(self, nodes):
        arr = np.ascontiguousarray(np.asarray(nodes, dtype=NODE_DTYPE))
        if arr.ndim != 1 or arr.size == 0:
            raise ArgumentError("encoded tree requires at least one node")
        self._nodes = arr
        self._nodes.setflags(write=False)
        cls = arr["class_id"]
        leaf = cls != NO_CLASS
        self._leaf_count = int(leaf.sum())
        self._internal = np.nonzero(~leaf)[0].astype(np.uint32)
        self._max_attribute = int(arr["attribute"].max())
        # depth by forward propagation; non-forward links skipped (tree.cpp:49-60)
        n = arr.size
        depth = np.zeros(n, dtype=np.int64)
        d = 0
        child = arr["child"]
        for i in range(n):
            if leaf[i]:
                d = max(d, int(depth[i]))
            else:
                c = int(child[i])
                if c > i and c + 1 < n:
                    depth[c] = depth[i] + 1
                    depth[c + 1] = depth[i] + 1
        self._depth = d
        self._handle = None
        self._handle_lock = threading.Lock()

    # --- reference accessors ------------------------------------------------
    def size(self) -> int:
        return int(self._nodes.size)

    def nodes(self) -> np.ndarray:
        return self._nodes

    def node(self, i: int):
        return self._nodes[i]

    def leaf_count(self) -> int:
        return self._leaf_count

    def depth(self) -> int:
        return self._depth

    def max_attribute(self) -> int:
        return self._max_attribute

    def internal_indices(self) -> np.ndarray:
        return self._internal

    def __len__(self) -> int:
        return self.size()

    def __eq__(self, other) -> bool:
        return isinstance(other, EncodedTree) and self._nodes.tobytes() == other._nodes.tobytes()

    # --- device handle (created lazily, owned by this object) ---------------
    def handle(self):
        """The native st_tree, created once (thread-safe: concurrent first
        calls must not create and then free competing handles)."""
        h = self._handle
        if h is None:
            with self._handle_lock:
                if self._handle is None:
                    from .evaluate import _TreeHandle

                    self._handle = _TreeHandle(self._nodes)
                h = self._handle
        return h


def encode_breadth_first(root: LinkedNode) -> EncodedTree:
    """Queue-driven BFS encoding (tree.cpp:72-113)."""
    queue = [(root, "root")]
    out = []
    child_counter = 1
    i = 0
    while i < len(queue):
        node, path = queue[i]
        has_l, has_r = node.left is not None, node.right is not None
        if has_l != has_r:
            raise StructureError(f"non-full node (exactly one child) at {path}")
        if node.is_leaf():
            if node.class_val is None:
                raise StructureError(f"leaf without a class at {path}")
            if node.class_val == NO_CLASS:
                raise StructureError(f"reserved class id at {path}")
            out.append((0, math.inf, i, node.class_val))
        else:
            if node.class_val is not None:
                raise StructureError(f"class on an internal node at {path}")
            out.append((node.attribute, node.threshold, child_counter, NO_CLASS))
            queue.append((node.left, path + ".left"))
            queue.append((node.right, path + ".right"))
            child_counter += 2
        i += 1
    return EncodedTree(np.array(out, dtype=NODE_DTYPE))


def decode(tree: EncodedTree) -> LinkedNode:
    """Rebuild the linked form (tree.cpp:117-136)."""
    nodes = tree.nodes()

    def at(i: int) -> LinkedNode:
        nd = nodes[i]
        if int(nd["class_id"]) != NO_CLASS:
            return make_leaf(int(nd["class_id"]))
        c = int(nd["child"])
        if c <= i or c + 1 >= tree.size():
            raise ArgumentError(f"node {i} has a non-BFS child link; cannot decode")
        return make_split(int(nd["attribute"]), float(nd["threshold"]), at(c), at(c + 1))

    return at(0)


@dataclass
class Diagnostic:
    node: int
    message: str


def validate(tree: EncodedTree) -> List[Diagnostic]:
    """Structural findings (tree.cpp:138-189); empty means well formed."""
    nodes = tree.nodes()
    n = tree.size()
    findings: List[Diagnostic] = []
    referenced = np.zeros(n, dtype=np.int64)
    for i in range(n):
        nd = nodes[i]
        if int(nd["class_id"]) != NO_CLASS:
            if int(nd["child"]) != i:
                findings.append(Diagnostic(i, f"leaf child index is {int(nd['child'])}, expected self-loop {i}"))
            if not float(nd["threshold"]) == math.inf:
                findings.append(Diagnostic(i, "leaf threshold is not +inf"))
        else:
            if not math.isfinite(float(nd["threshold"])):
                findings.append(Diagnostic(i, "internal threshold is not finite"))
            c = int(nd["child"])
            if c + 1 >= n:
                findings.append(Diagnostic(i, f"child index {c} out of range"))
            elif c <= i:
                findings.append(Diagnostic(i, f"non-BFS child link: child {c} does not point forward"))
            else:
                referenced[c] += 1
                referenced[c + 1] += 1
    if referenced[0] != 0:
        findings.append(Diagnostic(0, "root is referenced as a child"))
    for i in range(1, n):
        if referenced[i] == 0:
            findings.append(Diagnostic(i, "node is not referenced by any parent"))
        elif referenced[i] > 1:
            findings.append(Diagnostic(i, f"node is referenced {int(referenced[i])} times"))
    if n != 2 * tree.leaf_count() - 1:
        findings.append(Diagnostic(0, f"node count {n} != 2 * {tree.leaf_count()} - 1 (not a full tree)"))
    return findings


def processor_node_map(tree: EncodedTree) -> np.ndarray:
    """Lane -> internal node map (tree.cpp:204-209)."""
    return tree.internal_indices().copy()


# --------------------------------------------------------------------------
# Tree JSON schema v1 (io.hpp:19-31, io.cpp:156-263)
# --------------------------------------------------------------------------
def _u32(value, name, what, i):
    if isinstance(value, bool) or not isinstance(value, int) or value < 0 or value > 0xFFFFFFFF:
        raise SchemaError(f"{name}: node {i}: {what} must be an unsigned 32-bit integer")
    return value


def load_tree_json_text(text: str, name: str = "<memory>") -> EncodedTree:
    try:
        doc = json.loads(text)
    except (ValueError, json.JSONDecodeError) as e:
        raise SchemaError(f"{name}: invalid JSON: {e}") from None
    if not isinstance(doc, dict):
        raise SchemaError(f"{name}: top level must be an object")
    ver = doc.get("version")
    if isinstance(ver, bool) or not isinstance(ver, int):
        raise SchemaError(f"{name}: missing integer 'version'")
    if ver != 1:
        raise SchemaError(f"{name}: unsupported schema version {ver}, expected 1")
    items = doc.get("nodes")
    if not isinstance(items, list) or not items:
        raise SchemaError(f"{name}: 'nodes' must be a non-empty array")
    n = len(items)
    out = np.zeros(n, dtype=NODE_DTYPE)
    for i, item in enumerate(items):
        if not isinstance(item, dict) or not all(k in item for k in ("attr", "thr", "child", "class")):
            raise SchemaError(f"{name}: node {i} must be an object with attr, thr, child, class")
        attr = _u32(item["attr"], name, "attr", i)
        child = _u32(item["child"], name, "child", i)
        if child >= n:
            raise SchemaError(f"{name}: node {i}: child index {child} out of range")
        cls, thr = item["class"], item["thr"]
        if cls is None:
            if isinstance(thr, bool) or not isinstance(thr, (int, float)):
                raise SchemaError(f"{name}: node {i}: internal thr must be a number")
            tf = np.float32(thr)
            if not math.isfinite(float(thr)) or not np.isfinite(tf):
                raise SchemaError(f"{name}: node {i}: internal thr must be finite")
            if child + 1 >= n:
                raise SchemaError(f"{name}: node {i}: right child index {child + 1} out of range")
            out[i] = (attr, tf, child, NO_CLASS)
        else:
            c = _u32(cls, name, "class", i)
            if c == NO_CLASS:
                raise SchemaError(f"{name}: node {i}: class id {NO_CLASS} is reserved")
            if thr not in ("-inf", "inf", "+inf"):
                raise SchemaError(f"{name}: node {i}: leaf thr must be the string \"-inf\"")
            out[i] = (attr, math.inf, child, c)
    return EncodedTree(out)


def load_tree_json(path) -> EncodedTree:
    try:
        with open(path, "r") as f:
            text = f.read()
    except OSError:
        from .errors import IoError

        raise IoError(f"cannot open {path} for reading") from None
    return load_tree_json_text(text, str(path))


def tree_to_json(tree: EncodedTree) -> str:
    """Leaves serialise their threshold as "-inf" (io.cpp:242-263)."""
    items = []
    for nd in tree.nodes():
        if int(nd["class_id"]) != NO_CLASS:
            items.append({"attr": int(nd["attribute"]), "child": int(nd["child"]),
                          "class": int(nd["class_id"]), "thr": "-inf"})
        else:
            items.append({"attr": int(nd["attribute"]), "child": int(nd["child"]),
                          "class": None, "thr": float(nd["threshold"])})
    return json.dumps({"nodes": items, "version": 1}, indent=2, sort_keys=True) + "\n"
