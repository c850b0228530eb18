"""Run manifests for the artifacts the B200 tools write (reference schema: manifest.py:10-29).

A manifest records the command, its input and output paths, the seed, and a digest of the fully
resolved configuration: SHA-256 over the configuration serialised as canonical JSON (keys sorted,
no insignificant whitespace), so two runs with the same configuration carry the same digest
whatever the key order they were built in.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import asdict, dataclass

__all__ = ["config_digest", "RunManifest", "make_manifest"]


def config_digest(payload) -> str:
    blob = json.dumps(payload, sort_keys=True, separators=(",", ":")).encode()
    return hashlib.sha256(blob).hexdigest()


@dataclass(frozen=True)
class RunManifest:
    command: str
    inputs: object   # paths (list) or {role: path} (dict), as the writer recorded them
    outputs: object
    seed: int | None
    config_digest: str

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, doc: dict) -> "RunManifest":
        return cls(command=doc["command"], inputs=doc["inputs"], outputs=doc["outputs"],
                   seed=doc["seed"], config_digest=doc["config_digest"])


def make_manifest(command: str, config, inputs=None, outputs=None,
                  seed: int | None = None) -> RunManifest:
    """Manifest of one tool run; the digest covers `config` (the resolved arguments)."""
    return RunManifest(command, list(inputs or []), list(outputs or []), seed,
                       config_digest(config))
