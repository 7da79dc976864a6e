"""Top stall lines per kernel from `ncu -i X --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 25
i = 0
while i < len(rows):
    r = rows[i]
    if r and r[0] == "Kernel Name":
        name = r[1]
        h = rows[i + 1]
        idx = {k: j for j, k in enumerate(h)}
        j = i + 2
        data = []
        while j < len(rows) and rows[j] and rows[j][0] != "Kernel Name":
            data.append(rows[j]); j += 1
        i = j
        if want not in name:
            continue
        col = idx["Warp Stall Sampling (All Samples)"]
        tot = sum(int(d[col] or 0) for d in data)
        print("==", name[:90], "samples", tot)
        for d in sorted(data, key=lambda d: -int(d[col] or 0))[:ntop]:
            print("  ", d[0][-5:], d[col], d[1][:95])
    else:
        i += 1
