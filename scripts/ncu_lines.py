"""Summarise an `ncu --page source --csv --print-source cuda,sass` dump: warp-stall samples
per CUDA source line (top N) with the dominant stall reasons.

    ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python scripts/ncu_lines.py src.csv [N] [function-substring]
"""
import csv
import sys


def main(path, top=25, func=None):
    rows = list(csv.reader(open(path)))
    files, cur, hdr, fn = {}, None, None, ""
    for r in rows:
        if r and r[0] == "Function Name":
            fn = r[1]
            continue
        if func and func not in fn:
            continue
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and r and r[0] and r[0] != "Function Name" and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            try:
                n = int(d["Warp Stall Sampling (All Samples)"])
            except ValueError:
                continue
            stalls = {k[6:]: int(v) for k, v in zip(hdr, r)
                      if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
            files[(cur, int(r[0]))] = (n, r[1].strip()[:70], stalls)
    tot = sum(v[0] for v in files.values()) or 1
    print(f"total samples {tot}")
    for (f, ln), (n, src, st) in sorted(files.items(), key=lambda kv: -kv[1][0])[:top]:
        best = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        bs = " ".join(f"{k}:{v}" for k, v in best if v)
        print(f"{100*n/tot:5.1f}% {f}:{ln:<4} {src:<70} {bs}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25,
         sys.argv[3] if len(sys.argv) > 3 else None)
