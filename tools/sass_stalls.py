"""Top stall-sampled SASS instructions of an ncu source-page CSV (--page source --csv --print-source sass),
with a few lines of context before each: which barrier / instruction each warp role waits on."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 3
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
samp = [int(r[iS]) if r[iS].isdigit() else 0 for r in data]
print("total samples", sum(samp))
order = sorted(range(len(data)), key=lambda i: -samp[i])[:top_n]
for i in sorted(order):
    print("-----")
    for j in range(max(0, i - ctx), i + 1):
        print(str(samp[j]).rjust(5), data[j][0][-5:], data[j][1].strip()[:110])
