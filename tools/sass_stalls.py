"""Top stall-sampled SASS instructions of an ncu source-page CSV (--page source --csv --print-source sass),
with a few lines of context before each: which barrier / instruction each warp role waits on."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 3
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]


def why(r):  # the two largest stall reasons of an instruction
    v = sorted(((int(r[i]) if r[i].isdigit() else 0, hdr[i][6:]) for i in reasons), reverse=True)[:2]
    return " ".join(f"{n}:{k}" for k, n in v if k)
samp = [int(r[iS]) if r[iS].isdigit() else 0 for r in data]
print("total samples", sum(samp))
tot = {}
for r in data:
    for i in reasons:
        tot[hdr[i][6:]] = tot.get(hdr[i][6:], 0) + (int(r[i]) if r[i].isdigit() else 0)
print("by reason:", ", ".join(f"{k} {v}" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
order = sorted(range(len(data)), key=lambda i: -samp[i])[:top_n]
for i in sorted(order):
    print("-----")
    for j in range(max(0, i - ctx), i + 1):
        print(str(samp[j]).rjust(5), data[j][0][-5:], data[j][1].strip()[:90].ljust(90), why(data[j]) if j == i else "")
