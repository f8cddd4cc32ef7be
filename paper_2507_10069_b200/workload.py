"""Trace ingestion without the reference installed.

The canonical traces are generated once by the reference's own
workload.generate and written with its write_trace (JSON lines,
pkg/src/mmsim/core.py:235-301); they live in tests/golden/traces/.  On the
GPU box (no /root/reference) they are read here into duck-type
compatible records with the fields the hot path uses
(pkg/src/mmsim/core.py:50-97).  When mmsim is importable the reference's own
`Request` objects work unchanged.
"""
from __future__ import annotations

import json
from dataclasses import dataclass


@dataclass(frozen=True)
class ImageInput:  # core.py:50-61
    content_hash: str
    token_count: int
    pixels: tuple


@dataclass
class Request:  # core.py:64-97
    id: int
    arrival_time: float
    modality: str
    text_input_len: int
    images: tuple
    output_len: int
    priority_hint: bool = False
    prefix_id: int | None = None
    prefix_len: int = 0

    @property
    def image_token_count(self) -> int:
        return sum(img.token_count for img in self.images)

    @property
    def total_input_len(self) -> int:
        return self.text_input_len + self.image_token_count

    @property
    def is_multimodal(self) -> bool:
        return self.modality == "multimodal"


def request_from_dict(doc: dict) -> Request:  # mirrors core.py:258-274
    images = tuple(ImageInput(str(i["hash"]), int(i["token_count"]),
                              (int(i["pixels"][0]), int(i["pixels"][1])))
                   for i in doc.get("images", []))
    return Request(id=int(doc["id"]), arrival_time=float(doc["arrival_time"]),
                   modality=str(doc["modality"]), text_input_len=int(doc["text_input_len"]),
                   images=images, output_len=int(doc["output_len"]),
                   priority_hint=bool(doc.get("priority_hint", False)),
                   prefix_id=(int(doc["prefix_id"]) if doc.get("prefix_id") is not None
                              else None),
                   prefix_len=int(doc.get("prefix_len", 0)))


def read_trace(path: str) -> list[Request]:
    import gzip
    out = []
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt", encoding="utf-8") as fh:
        for line in fh:
            line = line.strip()
            if line:
                out.append(request_from_dict(json.loads(line)))
    return out
