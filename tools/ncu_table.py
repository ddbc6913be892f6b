"""Summarise an `ncu --csv --log-file` launch list (skips ncu's preamble lines)."""
import csv, io, sys
from collections import OrderedDict

def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    d = OrderedDict()
    for r in rows:
        e = d.setdefault(r["ID"], {"kernel": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"]})
        e[r["Metric Name"]] = r["Metric Value"]
    return d

if __name__ == "__main__":
    d = load(sys.argv[1])
    keys = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    for i, e in d.items():
        ks = keys or [k for k in e if k not in ("kernel", "grid", "block")]
        print(i, e["kernel"][:48], e["grid"], " ".join(f"{k.split('.')[0].split('__')[-1]}={e.get(k)}" for k in ks))
