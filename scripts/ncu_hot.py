"""Top SASS lines by warp-stall samples from `ncu -i X --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
i = 0
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name":
        name = rows[i][1]
        hdr = rows[i + 1]
        j = i + 2
        data = []
        while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
            if len(rows[j]) >= len(hdr) - 1:
                data.append(dict(zip(hdr, rows[j])))
            j += 1
        key = "Warp Stall Sampling (All Samples)"
        tot = sum(int(d[key] or 0) for d in data)
        print(f"== {name[:120]}  samples={tot}")
        for d in sorted(data, key=lambda d: -int(d[key] or 0))[:n]:
            print(f"{d[key]:>6} {d['Address'][-5:]} {d['Source'].strip()[:100]}")
        i = j
    else:
        i += 1
