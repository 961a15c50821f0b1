"""Summaries of ncu reports for profiles/ (dev helper)."""
import csv, subprocess, sys

def details(rep, keys):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    res = []
    for line in out.splitlines():
        r = line.strip().strip('"').split('","')
        if len(r) >= 4 and any(k in r[-3] for k in keys):
            res.append(f"{r[-4]} | {r[-3]} | {r[-2]} | {r[-1]}")
    return res

def source_top(rep, k=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None; lines = []; cur = None
    for r in rows:
        if r and r[0] == "File Path": cur = r[1]; continue
        if r and r[0] == "Line No": hdr = r; continue
        if hdr and r and r[0] and r[0] != "Function Name":
            try:
                ie = hdr.index("Instructions Executed"); ws = hdr.index("Warp Stall Sampling (All Samples)")
                lines.append((int(r[ie]), int(r[ws]), cur.split('/')[-1], r[0], r[1][:90]))
            except Exception:
                pass
    tot = sum(l[0] for l in lines) or 1; tots = sum(l[1] for l in lines) or 1
    res = [f"total warp instructions {tot}, stall samples {tots}"]
    for l in sorted(lines, reverse=True)[:k]:
        res.append(f"{l[0]:>12} {100*l[0]/tot:5.1f}% stall {100*l[1]/tots:5.1f}% {l[2]}:{l[3]}: {l[4]}")
    return res

if __name__ == "__main__":
    rep = sys.argv[1]
    keys = ["Duration", "Executed Ipc A", "Issue Slots Busy", "Warp Cycles Per Issued", "Achieved Occupancy",
            "Theoretical Occupancy", "Registers Per", "Avg. Active Threads", "Eligible Warps", "DRAM Throughput",
            "Compute (SM) Throughput", "Memory Throughput"]
    print("\n".join(details(rep, keys)))
    print("\n".join(source_top(rep, int(sys.argv[2]) if len(sys.argv) > 2 else 25)))
