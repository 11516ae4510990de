"""One-line-per-kernel summary of ncu --set full reports (tools/; profiles/ tables):
duration, DRAM read/write, DRAM %, tensor %, XU %, issue %."""
import csv
import io
import subprocess
import sys

KEYS = {
    "us": "gpu__time_duration.sum",
    "rd": "dram__bytes_read.sum",
    "wr": "dram__bytes_write.sum",
    "dram%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor%": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "xu%": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "issue%": "sm__inst_issued.avg.pct_of_peak_sustained_active",
}
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def summarize(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")[:60]}
        for k, m in KEYS.items():
            if m in hdr:
                i = hdr.index(m)
                v = float(r[i].replace(",", "")) if r[i] else float("nan")
                d[k] = v * SCALE.get(units[i], 1.0) if k in ("us", "rd", "wr") else v
        out.append(d)
    return out


if __name__ == "__main__":
    print("| kernel | us | DRAM read MB | DRAM write MB | DRAM % | tensor % | XU % | issue % |")
    print("|---|---|---|---|---|---|---|---|")
    for rep in sys.argv[1:]:
        for d in summarize(rep):
            f = lambda k: f"{d[k]:.1f}" if k in d else "-"
            print(f"| {d['kernel']} | {f('us')} | {f('rd')} | {f('wr')} | {f('dram%')} | {f('tensor%')} | {f('xu%')} | {f('issue%')} |")
