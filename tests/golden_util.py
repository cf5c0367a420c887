"""Helpers to read the golden fixtures (tests/golden/, produced by the reference)."""
import numpy as np


def unpad(prefix_rows, depths):
    return [list(map(int, prefix_rows[i, : depths[i]])) for i in range(len(depths))]


def pool_nodes(pools, name):
    pre = pools[f"{name}_nodes_prefix"]
    dep = pools[f"{name}_nodes_depth"]
    return unpad(pre, dep), pools[f"{name}_nodes_heads"], pools[f"{name}_nodes_lb"]


def pool_children(pools, name):
    par = unpad(pools[f"{name}_parents_prefix"], pools[f"{name}_parents_depth"])
    kids = unpad(pools[f"{name}_children_prefix"], pools[f"{name}_children_depth"])
    return (par, kids, pools[f"{name}_children_parent"], pools[f"{name}_children_heads"],
            pools[f"{name}_children_lb"])


def instance_p(instances, name):
    d = instances[name]
    return np.asarray(d["p"], np.int32).reshape(d["n"], d["m"])


CLASSES = ["ta001", "ta021", "ta051", "ta081", "ta101"]
