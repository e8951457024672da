"""Summarise an ncu --set full report of k_compress launches: per-tile instruction mix, pipe
utilisation, stall reasons and the share of stall samples inside / outside the tile body.
Usage: python tools/ncu_summary.py report.ncu-rep [tiles_per_launch]"""
import csv, collections, subprocess, sys

rep = sys.argv[1]
tiles = float(sys.argv[2]) if len(sys.argv) > 2 else 32 * 4096 * 4096 / 4096


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(run("--page", "raw", "--csv").splitlines()))
hdr, data = raw[0], raw[2:]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum"]
for d in data:
    print(d[hdr.index("Kernel Name")][:70])
    for w in want:
        print(f"  {w:70s} {d[hdr.index(w)]}")
    st = [(h, float(d[hdr.index(h)] or 0)) for h in hdr
          if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
    tot = sum(v for _, v in st) or 1
    st.sort(key=lambda x: -x[1])
    print("  stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {v / tot:.3f}" for h, v in st[:9]))

src = run("--page", "source", "--csv", "--print-source", "sass").split("\n")
blocks, cur = [], None
for l in src:
    if l.startswith('"Kernel Name"'):
        cur = [l]
        blocks.append(cur)
    elif cur is not None:
        cur.append(l)
for b in blocks:
    rows = list(csv.reader(b[1:]))
    h, rs = rows[0], [r for r in rows[1:] if len(rows[0]) == len(r)]
    iE, iS, iSm = h.index("Instructions Executed"), h.index("Source"), h.index("# Samples")
    ops, samp = collections.Counter(), collections.Counter()
    for r in rs:
        t = r[iS].strip().split()
        if not t:
            continue
        o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[o] += float(r[iE] or 0)
        samp[o] += float(r[iSm] or 0)
    idx = [i for i, r in enumerate(rs) if r[iS].strip().startswith(("LDS", "FFMA2", "FADD2"))]
    body_s = sum(float(r[iSm] or 0) for i, r in enumerate(rs) if idx and idx[0] <= i <= idx[-1]
                 and r[iS].strip().split()[0] not in ("SYNCS.PHASECHK.TRANS64.TRYWAIT",))
    tot_s = sum(samp.values()) or 1
    print(b[0][15:85])
    print(f"  instr/tile {sum(ops.values()) / tiles:.1f}; samples in body span {body_s / tot_s:.3f}")
    print("  ", sorted([(k, round(v / tiles, 1)) for k, v in ops.items() if v / tiles > 0.9], key=lambda x: -x[1]))
