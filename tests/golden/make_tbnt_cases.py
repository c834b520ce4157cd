"""Golden .tbnt error cases from the UNMODIFIED reference loader.

Run in the builder container (where /root/reference exists):

    python tests/golden/make_tbnt_cases.py

Takes the reference-written ``adult.tbnt`` stream, derives malformed variants
(truncations, bad magic / version / CRC, metadata the reference rejects or
accepts, size mismatches, invalid config values), re-seals the CRC where the
case is about the payload, and records which exception class the reference's
``tabserve.model.io.load_model`` (io.py:60-112) raises for each — or, for
accepted streams, the reference's own re-serialization.  Only the .npz travels;
tests/test_host.py replays the cases against the native parser (csrc/tbnt.cpp).
"""
from __future__ import annotations

import json
import struct
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, str(REF))
    from tabserve.model import io as RIO

    base = (OUT / "adult.tbnt").read_bytes()

    def sections(b):
        off, out = 6, []
        for _ in range(3):
            (n,) = struct.unpack_from("<I", b, off)
            out.append(b[off + 4:off + 4 + n])
            off += 4 + n
        return out

    def seal(meta: bytes, stats: bytes, flat: bytes, version: int = 1) -> bytes:
        body = b"TBNT" + struct.pack("<H", version)
        for p in (meta, stats, flat):
            body += struct.pack("<I", len(p)) + p
        return body + struct.pack("<I", RIO.crc32c(body))

    meta_b, stats_b, flat_b = sections(base)
    meta = json.loads(meta_b)

    def with_meta(**upd):
        m = json.loads(meta_b)
        for k, v in upd.items():
            if v is None:
                m.pop(k, None)
            else:
                m[k] = v
        return seal(json.dumps(m).encode(), stats_b, flat_b)

    def with_cfg(**upd):
        c = dict(meta["config"])
        for k, v in upd.items():
            if v is None:
                c.pop(k, None)
            else:
                c[k] = v
        return with_meta(config=c)

    cases = {
        "ok": base,
        "short": base[:9],
        "header_only": base[:12],
        "cut_mid_section": base[:300],
        "cut_crc": base[:-2],
        "magic": b"XXXX" + base[4:],
        "version2": base[:4] + struct.pack("<H", 2) + base[6:],
        "crc_flip": base[:100] + bytes([base[100] ^ 0xFF]) + base[101:],
        "trailing": base[:-4] + b"\0\0\0\0" + base[-4:],
        "meta_not_json": seal(b"{not json", stats_b, flat_b),
        "meta_no_config": with_meta(config=None),
        "cfg_unknown_key": with_cfg(dropout=0.1),
        "cfg_missing_F": with_cfg(feature_count=None),
        "cfg_bad_F": with_cfg(feature_count=0),
        "cfg_bad_gamma": with_cfg(gamma=0.5),
        "cfg_bad_classes": with_cfg(n_classes=1),
        "cfg_string": with_cfg(n_d="8"),
        "meta_pretty": seal(json.dumps(meta, indent=2, sort_keys=False).encode(), stats_b, flat_b),
        "stats_short": seal(meta_b, stats_b[:-8], flat_b),
        "flat_short": seal(meta_b, stats_b, flat_b[:-8]),
        "flat_long": seal(meta_b, stats_b, flat_b + b"\0" * 8),
        "empty_version": with_meta(model_version=""),
        "var_zero": seal(meta_b, stats_b[:len(stats_b) // 2] + b"\0" * (len(stats_b) // 2), flat_b),
        "unicode_version": with_meta(model_version="vérsion-☃"),
    }
    out = {}
    for name, b in cases.items():
        try:
            m = RIO.load_model(b)
            res = "ok"
            out[name + "__reserialized"] = np.frombuffer(RIO.save_model(m), dtype=np.uint8)
        except Exception as exc:        # noqa: BLE001 — we record the class
            res = type(exc).__name__
        out[name + "__stream"] = np.frombuffer(b, dtype=np.uint8)
        out[name + "__expect"] = np.array(res)
        print(f"{name:18s} -> {res}")
    np.savez_compressed(OUT / "tbnt_cases.npz", **out)


if __name__ == "__main__":
    main()
