"""Warp-stall samples per instruction range from an `ncu --page source --csv --print-source sass`
export (tools/exp/src_prof.sh writes one for the c3 ping-pong kernel).

    python tools/src_stalls.py gpurun_out/c3_source_sass.csv.gz             # totals + top 25 instructions
    python tools/src_stalls.py FILE name:a:b name:a:b ...                  # sample share per SASS index range
"""
import collections
import csv
import gzip
import sys


def load(path):
    f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    rows = list(csv.reader(f))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    ins = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        st = {h[6:]: int(r[ix[h]] or 0) for h in stalls}
        ins.append((r[ix["Source"]].strip(), int(r[ix["Warp Stall Sampling (All Samples)"]] or 0),
                    int(r[ix["Instructions Executed"]] or 0), st))
    return ins


def main():
    ins = load(sys.argv[1])
    tot = sum(i[1] for i in ins)
    agg = collections.Counter()
    for i in ins:
        agg.update(i[3])
    print(f"{len(ins)} SASS instructions, {tot} stall samples")
    print("all warps:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in agg.most_common(8)))
    if len(sys.argv) == 2:
        for k, (src, s, e, st) in sorted(enumerate(ins), key=lambda t: -t[1][1])[:25]:
            top = ", ".join(f"{a} {b}" for a, b in sorted(st.items(), key=lambda t: -t[1])[:2] if b)
            print(f"{k:5d} {100 * s / tot:5.2f}% exec {e:8d}  {src[:58]:58s} {top}")
        return
    for spec in sys.argv[2:]:
        name, a, b = spec.split(":")
        part = ins[int(a):int(b)]
        s = sum(i[1] for i in part)
        c = collections.Counter()
        for i in part:
            c.update(i[3])
        top = ", ".join(f"{k} {100 * v / max(s, 1):.0f}%" for k, v in c.most_common(4) if v)
        print(f"{name:22s} {100 * s / tot:5.1f}% of samples   {top}")


if __name__ == "__main__":
    main()
