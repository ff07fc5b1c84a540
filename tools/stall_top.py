"""Top SASS lines by warp-stall samples from an `ncu -i REP --page source --csv --print-source sass` dump
(not part of the library): python tools/stall_top.py SOURCE.csv [N] > profiles/<round>/ncu_stall_top_<cfg>.txt.
A dump may hold several kernels (a header row "Kernel Name" starts each)."""
import csv
import sys


def main():
    path = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    rows = list(csv.reader(open(path)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1] if len(r) > 1 else "?", "hdr": None, "data": []}
            blocks.append(cur)
        elif cur is not None and r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and cur["hdr"] and len(r) > 5:
            cur["data"].append(r)
    for b in blocks:
        h = b["hdr"]
        iS, iE, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
        data = [(int(r[iS] or 0), int(r[iE] or 0), r[iSrc].strip()) for r in b["data"] if r[iS].isdigit()]
        tot = sum(d[0] for d in data) or 1
        print(f"# ncu --set full source page (SASS), top {n} instructions by warp-stall samples; {b['name'][:110]}")
        print(f"# total samples {tot}")
        print("share  samples  executed  instruction")
        for s, e, src in sorted(data, key=lambda d: -d[0])[:n]:
            print(f"{s / tot:.3f} {s:8d} {e:11d}  {src[:90]}")
        print()


if __name__ == "__main__":
    main()
