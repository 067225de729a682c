"""ProfileArchive: the on-disk JSON format for join results (archive.hpp:13-49).

Schema version 1. +inf encodes as the string "inf" and undefined indexes as -1;
floats are written at full round-trip precision (repr), so write -> read is the
identity on every field (SPEC.md io module: "lossless round-trip including
sentinels"). The input data can be embedded (the keep-data contract,
archive.hpp:24-25). Positions are 0-based in the archive; the printed summary
block is 1-based (archive.hpp:51-54).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import MatrixProfile

SCHEMA_VERSION = 1


class ArchiveError(ValueError):
    """Corrupt payload or unsupported schema (the reference's IoError, error.hpp:28-32)."""


def _enc(v: float):
    if math.isinf(v) and v > 0:
        return "inf"
    if math.isnan(v):
        raise ArchiveError("NaN has no archive encoding")
    return float(v)


def _dec(v) -> float:
    if v == "inf":
        return math.inf
    if isinstance(v, (int, float)):
        return float(v)
    raise ArchiveError(f"bad float payload {v!r}")


@dataclass
class ProfileArchive:
    """Mirror of mprof::ProfileArchive (archive.hpp:17-46) for the join result."""
    profile: MatrixProfile
    mode: str = "stomp"
    ez_fraction: float = 0.5
    data_a: Optional[np.ndarray] = None
    data_b: Optional[np.ndarray] = None
    name_a: str = ""
    name_b: str = ""
    source_a: str = ""
    source_b: str = ""
    extra: dict = field(default_factory=dict)  # discovery results bolted on later

    def window(self) -> int:
        return self.profile.window

    def exclusion_zone(self) -> int:
        return self.profile.exclusion_zone

    def profile_size(self) -> int:
        return self.profile.size()

    def coverage(self) -> float:
        return self.profile.coverage

    def is_ab(self) -> bool:
        return self.profile.join_kind == "ab"


def archive_to_json(ar: ProfileArchive) -> str:
    p = ar.profile
    doc = {
        "schema_version": SCHEMA_VERSION,
        "mode": ar.mode or p.mode,
        "join_kind": p.join_kind,
        "window": int(p.window),
        "exclusion_zone": int(p.exclusion_zone),
        "ez_fraction": ar.ez_fraction,
        "coverage": float(p.coverage),
        "seed": int(p.seed),
        "data_len": int(p.data_len),
        "data_len_b": int(p.data_len_b),
        "data_dims": int(p.data_dims),
        "profile_size": int(p.size()),
        "values": [_enc(v) for v in np.asarray(p.values, dtype=np.float64).tolist()],
        "index": np.asarray(p.index, dtype=np.int64).tolist(),
        "left_index": np.asarray(p.left_index, dtype=np.int64).tolist() if p.has_left_right() else None,
        "right_index": np.asarray(p.right_index, dtype=np.int64).tolist() if p.has_left_right() else None,
        "data_a": None if ar.data_a is None else [float(v) for v in np.asarray(ar.data_a).tolist()],
        "data_b": None if ar.data_b is None else [float(v) for v in np.asarray(ar.data_b).tolist()],
        "name_a": ar.name_a, "name_b": ar.name_b,
        "source_a": ar.source_a, "source_b": ar.source_b,
        "extra": ar.extra,
    }
    return json.dumps(doc, allow_nan=False)


def archive_from_json(text: str) -> ProfileArchive:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise ArchiveError(f"corrupt archive: {e}") from None
    if doc.get("schema_version") != SCHEMA_VERSION:
        raise ArchiveError(f"unsupported schema_version {doc.get('schema_version')!r}")
    try:
        values = np.array([_dec(v) for v in doc["values"]], dtype=np.float64)
        index = np.array(doc["index"], dtype=np.int64)
        if values.size != index.size or values.size != doc["profile_size"]:
            raise ArchiveError("profile length mismatch")
        lr = doc.get("left_index") is not None
        prof = MatrixProfile(
            values=values, index=index,
            left_index=np.array(doc["left_index"], dtype=np.int64) if lr else np.empty(0, np.int64),
            right_index=np.array(doc["right_index"], dtype=np.int64) if lr else np.empty(0, np.int64),
            window=int(doc["window"]), exclusion_zone=int(doc["exclusion_zone"]),
            mode=doc["mode"], join_kind=doc["join_kind"], coverage=float(doc["coverage"]),
            seed=int(doc["seed"]), data_len=int(doc["data_len"]), data_len_b=int(doc["data_len_b"]),
            data_dims=int(doc["data_dims"]))
    except (KeyError, TypeError, ValueError) as e:
        raise ArchiveError(f"corrupt archive: {e}") from None
    return ProfileArchive(
        profile=prof, mode=doc["mode"], ez_fraction=float(doc["ez_fraction"]),
        data_a=None if doc.get("data_a") is None else np.array(doc["data_a"], dtype=np.float64),
        data_b=None if doc.get("data_b") is None else np.array(doc["data_b"], dtype=np.float64),
        name_a=doc.get("name_a", ""), name_b=doc.get("name_b", ""),
        source_a=doc.get("source_a", ""), source_b=doc.get("source_b", ""),
        extra=doc.get("extra", {}))


def write_profile(ar: ProfileArchive, path: str) -> None:
    try:
        with open(path, "w") as f:
            f.write(archive_to_json(ar))
    except OSError as e:
        raise ArchiveError(f"cannot write {path}: {e}") from None


def read_profile(path: str) -> ProfileArchive:
    try:
        with open(path) as f:
            return archive_from_json(f.read())
    except OSError as e:
        raise ArchiveError(f"cannot read {path}: {e}") from None


def render_profile_block(ar: ProfileArchive) -> str:
    """Printed summary (archive.hpp:51-54); positions 1-based."""
    p = ar.profile
    fin = np.isfinite(p.values)
    lines = [
        f"Matrix profile ({ar.mode}, {'AB-join' if ar.is_ab() else 'self-join'})",
        f"Profile size = {p.size()}",
        f"Window size = {p.window}",
        f"Exclusion zone = {p.exclusion_zone}",
        f"Coverage = {p.coverage:g}",
    ]
    if fin.any():
        i_min = int(np.argmin(np.where(fin, p.values, np.inf)))
        i_max = int(np.argmax(np.where(fin, p.values, -np.inf)))
        lines.append(f"Min distance = {p.values[i_min]:.6g} at {i_min + 1} (nearest {p.index[i_min] + 1})")
        lines.append(f"Max distance = {p.values[i_max]:.6g} at {i_max + 1}")
    return "\n".join(lines) + "\n"
