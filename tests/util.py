"""Shared helpers for the parity tests (sequence encodings, fixture decoding)."""
import numpy as np


def from_pm(s: str) -> np.ndarray:
    return np.array([1 if ch == "+" else -1 for ch in s], np.int8)


def to_pm(a) -> str:
    return "".join("+" if int(x) > 0 else "-" for x in a)


def hx(x: float) -> str:
    return float(x).hex()


def unhex(s: str) -> float:
    return float.fromhex(s)
