#!/usr/bin/env python
"""Golden .tns cases from the REFERENCE parser (run here, where
/root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_tns_golden.py

Writes tests/golden/tns_cases.json: each case's text, parse options and the
reference's result (indices, values as float hex, shape, LoadStats) or its
exception type + message.  Checked by tests/test_host_api.py (host parser) and
tests/test_gpu.py (GPU parser)."""
import io
import json
import os
import random

import numpy as np
from shardkrp.tensor import parse_tns

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    rng = random.Random(7)
    out = []

    def rnd_text(nlines, nm, crlf=False, comments=True, blank=True, tail_nl=True, fmt="%.17g", dup=False):
        rows = []
        seen = set()
        for _ in range(nlines):
            while True:
                c = tuple(rng.randint(1, 40) for _ in range(nm))
                if dup or c not in seen:
                    break
            seen.add(c)
            v = rng.choice([rng.random(), rng.uniform(-1e6, 1e6), rng.random() * 1e-300, 0.0, 1e300 * rng.random()])
            rows.append(" ".join(map(str, c)) + (rng.choice([" ", "\t", "  "])) + (fmt % v))
        lines = []
        if comments:
            lines.append("# generated")
            lines.append("# shape: " + " ".join(["40"] * nm))
        for r in rows:
            if blank and rng.random() < 0.05:
                lines.append("   ")
            if comments and rng.random() < 0.03:
                lines.append("# note")
            lines.append(("  " if rng.random() < 0.1 else "") + r)
        sep = "\r\n" if crlf else "\n"
        return sep.join(lines) + (sep if tail_nl else "")

    out.append(dict(name="kat_spec", text="2 1 3 1.5\n"))
    out.append(dict(name="kat_coalesce", text="1 1 1 2.0\n1 1 1 3.0\n", coalesce=True))
    out.append(dict(name="dup_rejected", text="1 1 1 2.0\n1 1 1 3.0\n"))
    out.append(dict(name="rand3", text=rnd_text(400, 3)))
    out.append(dict(name="rand4_crlf", text=rnd_text(300, 4, crlf=True)))
    out.append(dict(name="rand3_nocomment_notail", text=rnd_text(200, 3, comments=False, tail_nl=False)))
    out.append(dict(name="rand5_repr", text=rnd_text(200, 5, fmt="%r")))
    out.append(dict(name="rand3_f32", text=rnd_text(200, 3), dtype="float32"))
    out.append(dict(name="rand3_dups", text=rnd_text(300, 3, dup=True), coalesce=True))
    out.append(dict(name="explicit_shape", text="1 2 3 4.0\n", shape=[5, 5, 5]))
    out.append(dict(name="specials", text="1 1 1 inf\n1 1 2 -Infinity\n1 2 1 nan\n2 1 1 1_000.5\n2 2 2 +.5e-3\n"
                                          "3 3 3 123456789012345678901234567890e-10\n3 1 2 4.9e-324\n"
                                          "3 2 1 2.4703282292062328e-324\n"))
    out.append(dict(name="int_forms", text="+1 01 1_0 1.0\n2 2 2 2\n"))
    out.append(dict(name="err_few_cols", text="# c\n1 1 1.0\n"))
    out.append(dict(name="err_inconsistent", text="1 1 1 1.0\n\n1 1 2\n"))
    out.append(dict(name="err_nonnumeric_idx", text="1 1 1 1.0\n1 x 1 2.0\n"))
    out.append(dict(name="err_nonnumeric_val", text="1 1 1 1.0\n1 2 1 abc\n"))
    out.append(dict(name="err_zero_index", text="1 1 1 1.0\n0 2 1 2.0\n"))
    out.append(dict(name="err_no_data", text="# only comments\n\n"))
    out.append(dict(name="err_empty", text=""))
    out.append(dict(name="err_bad_header_before", text="# shape: a b c\n1 1 1 1.0\n"))
    out.append(dict(name="err_out_of_bounds", text="# shape: 2 2 2\n3 1 1 1.0\n"))
    return out


def main():
    res = []
    for c in cases():
        kw = dict(coalesce_duplicates=c.get("coalesce", False))
        if c.get("shape"):
            kw["shape"] = tuple(c["shape"])
        if c.get("dtype"):
            kw["value_dtype"] = np.dtype(c["dtype"])
        try:
            t = parse_tns(io.StringIO(c["text"]), **kw)
            c["result"] = dict(indices=t.indices.astype(np.int64).tolist(),
                               values=[float(v).hex() for v in t.values.astype(np.float64)],
                               dtype=str(t.values.dtype), shape=list(t.shape),
                               stats=dict(nnz=t.stats.nnz, zero_values=t.stats.zero_values,
                                          duplicates=t.stats.duplicates, coalesced=t.stats.coalesced))
        except Exception as exc:  # noqa: BLE001 - the exception IS the expected output
            c["error"] = dict(type=type(exc).__name__, message=str(exc))
        res.append(c)
    with open(os.path.join(HERE, "tns_cases.json"), "w") as fh:
        json.dump(res, fh)
    print(len(res), "cases")


if __name__ == "__main__":
    main()
