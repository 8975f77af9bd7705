"""Summarise an `ncu --page source --csv --print-source sass` export: top SASS lines by warp
stall samples with their dominant stall reasons, plus stall totals (dev tool)."""
import csv
import sys


def main(path, top=45):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {h: 0 for h in stall_cols}
    allsamp = 0
    recs = []
    for n, r in enumerate(data):
        if len(r) < len(hdr):
            continue
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        allsamp += s
        st = {h: int(r[ix[h]] or 0) for h in stall_cols}
        for h in stall_cols:
            tot[h] += st[h]
        recs.append((s, n, r[ix["Source"]].strip(), st, int(r[ix["Instructions Executed"]] or 0)))
    print(f"total samples {allsamp}")
    for h, v in sorted(tot.items(), key=lambda kv: -kv[1])[:12]:
        print(f"  {h:24s} {v:8d} {100.0 * v / max(allsamp, 1):5.1f}%")
    print()
    for s, n, src, st, ex in sorted(recs, key=lambda x: -x[0])[:top]:
        top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        t = " ".join(f"{k[6:]}={v}" for k, v in top3 if v)
        print(f"{n:5d} {s:6d} {100.0 * s / allsamp:5.1f}%  ex={ex:9d}  {src[:60]:60s} {t}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 45)
