"""Summarise an ncu --set full report of k_compress launches: per-tile instruction mix, pipe
utilisation, stall reasons and the share of stall samples inside / outside the tile body.
Usage: python tools/ncu_summary.py report.ncu-rep [tiles_per_launch] [--traffic-json out.json]
(--traffic-json writes the DRAM bytes per pixel of every k_compress / k_forward launch, the file
bench.py reads for roofline.traffic)."""
import csv, collections, subprocess, sys

import json

args = [a for a in sys.argv[1:]]
tj = None
if "--traffic-json" in args:
    i = args.index("--traffic-json")
    tj = args[i + 1]
    del args[i:i + 2]
rep = args[0]
tiles = float(args[1]) if len(args) > 1 else 32 * 4096 * 4096 / 4096


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

if tj:
    px = tiles * 4096
    per = {}
    for d in data:
        name = d[hdr.index("Kernel Name")]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(d[hdr.index("dram__bytes_read.sum")]) * scale[raw[1][hdr.index("dram__bytes_read.sum")]]
        wr = float(d[hdr.index("dram__bytes_write.sum")]) * scale[raw[1][hdr.index("dram__bytes_write.sum")]]
        inst = float(d[hdr.index("smsp__inst_executed.sum")])
        per[name] = {"dram_bytes_per_px": (rd + wr) / px, "read_per_px": rd / px, "write_per_px": wr / px,
                     "warp_instr_per_tile": inst / tiles,
                     "issue_active_pct": float(d[hdr.index("smsp__issue_active.avg.pct_of_peak_sustained_active")])}
    comp = [v["dram_bytes_per_px"] for k, v in per.items() if "k_compress" in k]
    with open(tj, "w") as f:
        json.dump({"source": f"ncu --set full, {int(tiles)} tiles of 4 KiB per launch "
                             f"(summary: profiles/r02_ncu_full_summary.txt)",
                   "dram_bytes_per_px": sum(comp) / max(1, len(comp)), "per_kernel": per}, f, indent=1)

src = run("--page", "source", "--csv", "--print-source", "sass").split("\n")
blocks, cur = [], None
for l in src:
    if l.startswith('"Kernel Name"'):
        cur = [l]
        blocks.append(cur)
    elif cur is not None:
        cur.append(l)
seen = set()
for b in blocks:
    if b[0] in seen:  # the source page lists each kernel once per view
        continue
    seen.add(b[0])
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
