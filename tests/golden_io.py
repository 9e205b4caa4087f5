"""Loader for the reference-generated fixtures in tests/golden (see tools/make_golden.py)."""
import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(group: str) -> dict:
    raw = np.load(os.path.join(GOLDEN, f"{group}.npz"), allow_pickle=False)
    cases = {}
    for name in raw["__cases"]:
        name = str(name)
        prefix = name + "__"
        case = {}
        for key in raw.files:
            if key.startswith(prefix):
                val = raw[key]
                case[key[len(prefix):]] = val.item() if val.ndim == 0 else val
        cases[name] = case
    return cases


def sha(data) -> str:
    return hashlib.sha256(np.ascontiguousarray(data).tobytes()).hexdigest()


def codes_for(case) -> np.ndarray:
    """Regenerate the fixture's genotype codes (reference numpy draws)."""
    import oracle
    if case.get("all_missing", False):
        return np.full((case["n"], case["p"]), 1, np.uint8)
    return oracle.random_codes(case["n"], case["p"], case["seed"],
                               missing_rate=case.get("missing", 0.0))
