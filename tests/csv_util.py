"""CSV helpers for the ingest tests: detail::write_csv_cell semantics
(table.hpp:180-193) and random byte soups over the reader's special bytes."""
import paper_2403_05821_b200 as po


def csv_cell(c: bytes) -> bytes:
    if c and not any(x in c for x in (b",", b'"', b"\r", b"\n")):
        return c
    return b'"' + c.replace(b'"', b'""') + b'"'


def to_csv(t, eol=b"\n") -> bytes:
    out = [b",".join(csv_cell(t.field_name(f)) for f in range(t.field_count()))]
    for r in range(t.row_count()):
        out.append(b",".join(csv_cell(t.cell(r, f)) for f in range(t.field_count())))
    return eol.join(out) + eol


def outcome(fn, data):
    try:
        t = fn(data)
        return ("ok", t.field_names, [t.row(r) for r in range(t.row_count())])
    except po.PrefixoptError as e:
        return (type(e).__name__, str(e))


SOUPS = [b'ab,"\n', b'ab,"\r\n', b'a,""\r\n\n x', b'x,y\n', b'"\n\r,', bytes(range(40))]
