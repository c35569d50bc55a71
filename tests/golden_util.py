"""Helpers shared by the parity tests (test infrastructure)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def random_instance(n_a: int, n_b: int, seed: int) -> np.ndarray:
    """test_util.hpp:19-30 random_instance: row-major u01 from mt19937_64(seed)."""
    from oracle.pyoracle import Oracle
    raw = Oracle.get().raw_stream(seed, n_a * n_b)
    return ((raw >> np.uint64(11)).astype(np.float64) * 2.0**-53).reshape(n_a, n_b)


def load_arrays(key: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"assign_{key}.npz")) as z:
        return {k: z[k] for k in z.files}


def pins_of(match_of_a, y_a, y_b, free_counts, phases, sum_ni, cost) -> dict:
    from oracle.pyoracle import fnv1a64
    return {
        "phases": int(phases), "sum_ni": int(sum_ni), "cost_hex": float(cost).hex(),
        "fnv_match": "%016x" % fnv1a64(np.asarray(match_of_a, np.int32)),
        "fnv_duals": "%016x" % fnv1a64(np.concatenate([np.asarray(y_a, np.int64),
                                                        np.asarray(y_b, np.int64)])),
        "fnv_free": "%016x" % fnv1a64(np.asarray(free_counts, np.int64)),
    }


PIN_KEYS = ("phases", "sum_ni", "cost_hex", "fnv_match", "fnv_duals", "fnv_free")
