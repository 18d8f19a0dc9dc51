"""JSONL ingest (po_load_jsonl: host code behind the C ABI, csrc/jsonl.cpp)
against the reference's own load_jsonl (oracle/_ref, table.hpp:225-269):
same table, or same error class and message, on hand-written documents over
every JSON value kind, on random line soups over JSON's special bytes
(including invalid UTF-8), and on generated tables. Host-only: runs in the
CPU suite (the library loads without a GPU; this entry point uses none)."""
import json
import random

import pytest

import paper_2403_05821_b200 as po
from csv_util import outcome
from oracle.pyoracle import available, oracle
from paper_2403_05821_b200 import gen

pytestmark = pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built")

KNOWN = [
    b"", b"\n", b"\r\n", b"{}\n", b"{}", b'{"a":1}', b'{"a":"x"}\n{"b":"y"}\n',
    b'{"a":"x","b":2}\n\n{"b":3,"c":null}\r\n{"a":true,"d":false}',
    b'{"n":[1,2,{"x":"y"}],"o":{"k":[]}, "s":"q\\"u\\\\o\\/te"}\n',
    b'{"f":1.0,"g":1e5,"h":-0,"i":123456789012345678901234567890,"j":0.1,"k":1E-7,"l":-2.50}\n',
    b'{"u":"\\u00e9\\ud83d\\ude00\\n\\t\\u0001","v":"\xc3\xa9 raw"}\n',
    b'{"dup":"first","dup":"second","z":1}\n',
    b'{"a":1}\n[1,2]\n', b'{"a":1}\n"str"\n', b'{"a":1}\nnull\n', b'{"a":1}\n{"a":\n',
    b'{"a":1} trailing\n', b'{"":1}\n', b'{"a":"\xff"}\n', b'{"a":"\xc3"}\n', b"  {\"a\" : 1 }  \n",
    b'{"a":1}\n   \n', b'\t\n{"a":1}\n', b'{"a":"x\ny"}\n', b'{"a":1}\r\r\n',
]

SPECIAL = b'{}[]":,\\ \t\r\nabc01-.eE+tfnul\xc3\xa9\xff\x00\x1f'


def test_jsonl_known_documents():
    R = oracle("reference")
    for d in KNOWN:
        assert outcome(po.load_jsonl, d) == outcome(R.load_jsonl, d), d


def test_jsonl_line_soups():
    rng = random.Random(2024)
    R = oracle("reference")
    for _ in range(600):
        lines = []
        for _ in range(rng.randint(0, 4)):
            if rng.random() < 0.5:  # mostly valid objects with odd values
                obj = {rng.choice(["a", "b", "c", "é", "x y"]):
                       rng.choice([None, True, 1.5, -3, "s\n\"", [1, {"k": None}], {"z": "w"}, ""])
                       for _ in range(rng.randint(0, 3))}
                lines.append(json.dumps(obj, ensure_ascii=rng.random() < 0.5).encode())
            else:
                lines.append(bytes(rng.choice(SPECIAL) for _ in range(rng.randint(0, 12))))
        d = rng.choice([b"\n", b"\r\n"]).join(lines) + rng.choice([b"", b"\n"])
        assert outcome(po.load_jsonl, d) == outcome(R.load_jsonl, d), d


def test_jsonl_generated_table():
    t = gen.generate(1, n_rows=2000)
    names = [n.decode() for n in t.field_names]
    lines = []
    for r in range(t.row_count()):
        row = {names[f]: t.cell(r, f).decode("utf-8", "replace") for f in range(len(names))
               if (r + f) % 5}  # sparse rows: absent keys -> ""
        lines.append(json.dumps(row, ensure_ascii=False).encode())
    d = b"\n".join(lines) + b"\n"
    R = oracle("reference")
    assert outcome(po.load_jsonl, d) == outcome(R.load_jsonl, d)
