"""Shared helpers for the test suite."""
import numpy as np


def layer_from_case(case):
    """Package QuantizedLayer built from a golden case's arrays."""
    import paper_2512_17970_b200 as cg

    cfg = cg.QuantConfig(v=case["v"], m=case["m"], b=case["b"], g=case["g"])
    return cg.QuantizedLayer(
        case["rows"], case["cols"], cfg, cg.ScalePlane(case["scales"].copy()),
        tuple(cg.CodePlane(c.copy()) for c in case["codes"]),
        tuple(cg.Codebook(b.copy()) for b in case["books"]),
    )


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def tolerance_report(y, y_ref):
    """The three output checks of DESIGN.md §5."""
    y = np.asarray(y, np.float64)
    ref = np.asarray(y_ref, np.float64)
    scale = float(np.max(np.abs(ref))) or 1.0
    max_abs = float(np.max(np.abs(y - ref))) / scale
    rel_l2 = float(np.linalg.norm(y - ref) / (np.linalg.norm(ref) or 1.0))
    big = np.abs(ref) >= 1e-2 * scale
    per_el = float(np.max(np.abs(y - ref)[big] / np.abs(ref)[big])) if big.any() else 0.0
    return {"norm_max_abs": max_abs, "rel_l2": rel_l2, "max_rel_big": per_el}


# tolerance written in the test (north star: fp32-accumulate tolerance,
# max rel err <= 1e-2 vs the fp32 reference; SPEC.md:489 rel-L2 <= 1e-3)
TOL_NORM_MAX_ABS = 1e-3
TOL_REL_L2 = 1e-3
TOL_MAX_REL_BIG = 1e-2


def assert_within_tolerance(y, y_ref, what=""):
    rep = tolerance_report(y, y_ref)
    assert rep["norm_max_abs"] <= TOL_NORM_MAX_ABS, (what, rep)
    assert rep["rel_l2"] <= TOL_REL_L2, (what, rep)
    assert rep["max_rel_big"] <= TOL_MAX_REL_BIG, (what, rep)
    return rep
