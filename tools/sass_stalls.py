"""Summarise an ncu source page (SASS, --csv) export: stall reasons overall
and by opcode class, instruction mix.  python tools/sass_stalls.py file.csv[.gz]"""
import collections
import csv
import gzip
import io
import sys


def main(path):
    f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    rows = list(csv.reader(f))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    by_op = collections.defaultdict(collections.Counter)
    inst = collections.Counter()
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        op = r[ix["Source"]].strip().split()[0] if r[ix["Source"]].strip() else "?"
        if op.startswith("@"):
            op = r[ix["Source"]].strip().split()[1]
        opc = op.split(".")[0]
        inst[opc] += int(r[ix["Instructions Executed"]] or 0)
        for s in stalls:
            v = int(r[ix[s]] or 0)
            tot[s] += v
            by_op[opc][s] += v
    n = sum(tot.values())
    print(f"samples {n}")
    for s, v in tot.most_common(10):
        print(f"  {s:28s} {100 * v / n:5.1f} %")
    print("samples by opcode:")
    ops = sorted(by_op, key=lambda o: -sum(by_op[o].values()))
    for o in ops[:14]:
        c = by_op[o]
        m = sum(c.values())
        top = ", ".join(f"{k[6:]} {100 * v / m:.0f}%" for k, v in c.most_common(3))
        print(f"  {o:10s} {100 * m / n:5.1f} %  (executed {inst[o]:.3e})  {top}")
    tot_i = sum(inst.values())
    print("instruction mix:", ", ".join(f"{o} {100 * v / tot_i:.1f}%" for o, v in inst.most_common(10)))


if __name__ == "__main__":
    main(sys.argv[1])
