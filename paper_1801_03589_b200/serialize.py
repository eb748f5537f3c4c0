"""Save / load the host inputs of a plan.

The reference rebuilds its tree and operators for every run (SPEC.md:335:
no persistence).  Here the tree (``TreeArrays`` + permutation + points) and
the operator tables (``OperatorTables``: fits, C, B, unique D, their index,
quadrants, leaf geometry) go to ONE compressed-free ``.npz``; loading it
skips the tree build and the table assembly (3.4 s + 0.2 s at N = 2M on the
GPU box) and gives bit-identical arrays, so the plan and every product are
bit-identical too.  Near / V / U blocks are not stored: plans built from
tables assemble them on the device in well under a second.
"""

from __future__ import annotations

import dataclasses

import numpy as np

from .operators import NesaParams, OperatorTables
from .quadtree import Tree, TreeArrays, TreeParams

__all__ = ["save_problem", "load_problem"]

_FORMAT = 1


def _dict_to_arrays(d: dict) -> tuple[np.ndarray, np.ndarray]:
    keys = np.array(sorted(d), dtype=np.int64)
    return keys, np.array([d[k] for k in keys], dtype=np.int64)


def save_problem(path: str, tree: Tree, tables: OperatorTables | None = None) -> None:
    """Write tree (and optionally tables) to ``path`` (.npz)."""
    a = tree.arrays
    out = {"format": np.array(_FORMAT)}
    for f in dataclasses.fields(TreeArrays):
        v = getattr(a, f.name)
        if isinstance(v, dict):
            out[f"t_{f.name}_k"], out[f"t_{f.name}_v"] = _dict_to_arrays(v)
        else:
            out[f"t_{f.name}"] = np.asarray(v)
    out["t_meta"] = np.array([tree.l0, tree.L], dtype=np.int64)
    out["t_root"] = np.array([tree.root_origin[0], tree.root_origin[1], tree.root_side])
    out["t_params"] = np.array([tree.params.P, tree.params.l0_groups_longest], dtype=np.int64)
    out["t_perm"] = np.asarray(tree.perm)
    out["t_points"] = np.asarray(tree.points)
    if tables is not None:
        p = tables.params
        out["o_params"] = np.array([p.Q, p.oversampling, p.rho_out_aux, p.rho_out_check,
                                    p.rho_in_check, p.rho_in_aux, p.pinv_cutoff])
        for name in ("out_fit", "in_fit"):
            d = getattr(tables, name)
            out[f"o_{name}_levels"] = np.array(sorted(d), dtype=np.int64)
            out[f"o_{name}"] = np.stack([d[k] for k in sorted(d)])
        for name in ("C", "B", "D", "d_keys", "d_index", "quad", "leaf_center", "leaf_h"):
            out[f"o_{name}"] = np.asarray(getattr(tables, name))
    np.savez(path, **out)


def load_problem(path: str) -> tuple[Tree, OperatorTables | None]:
    """Read what ``save_problem`` wrote: (tree, tables or None)."""
    z = np.load(path, allow_pickle=False)
    if int(z["format"]) != _FORMAT:
        raise ValueError(f"unsupported problem file format {int(z['format'])}")
    kw = {}
    for f in dataclasses.fields(TreeArrays):
        if f"t_{f.name}_k" in z:
            kw[f.name] = {int(k): int(v) for k, v in zip(z[f"t_{f.name}_k"], z[f"t_{f.name}_v"])}
        else:
            kw[f.name] = z[f"t_{f.name}"]
    arrays = TreeArrays(**kw)
    l0, L = (int(x) for x in z["t_meta"])
    ro = z["t_root"]
    tp = z["t_params"]
    tree = Tree(params=TreeParams(P=int(tp[0]), l0_groups_longest=int(tp[1])), l0=l0, L=L,
                root_origin=(float(ro[0]), float(ro[1])), root_side=float(ro[2]), arrays=arrays,
                perm=z["t_perm"], points=z["t_points"])
    tables = None
    if "o_params" in z:
        op = z["o_params"]
        params = NesaParams(Q=int(op[0]), oversampling=int(op[1]), rho_out_aux=float(op[2]),
                            rho_out_check=float(op[3]), rho_in_check=float(op[4]),
                            rho_in_aux=float(op[5]), pinv_cutoff=float(op[6]))
        fits = {}
        for name in ("out_fit", "in_fit"):
            fits[name] = {int(lv): m for lv, m in zip(z[f"o_{name}_levels"], z[f"o_{name}"])}
        tables = OperatorTables(params=params, out_fit=fits["out_fit"], in_fit=fits["in_fit"],
                                C=z["o_C"], B=z["o_B"], D=z["o_D"], d_keys=z["o_d_keys"],
                                d_index=z["o_d_index"], quad=z["o_quad"],
                                leaf_center=z["o_leaf_center"], leaf_h=z["o_leaf_h"])
    return tree, tables
