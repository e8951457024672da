"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file X) into
kernel | launches | mean us | share of the summed kernel time.
Usage: python tools/launch_summary.py launches.csv "<command it was captured from>" """
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
t = collections.defaultdict(list)
for r in rows:
    if r[12] == "gpu__time_duration.sum":
        v = float(r[14].replace(",", ""))
        t[r[4]].append(v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[13]])
tot = sum(sum(v) for v in t.values())
print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised) of\n# {sys.argv[2] if len(sys.argv) > 2 else ''}")
print("# kernel | launches | mean us | share of summed kernel time")
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / tot:.4f}")
# the bench's timed step is the 8 k_compress<r> passes + k_psnr; the other kernels are its secondary
# lines (fused sweep, Parseval sweep), timed separately
step = {k: v for k, v in t.items() if "k_compress<" in k or "k_psnr" in k}
st = sum(sum(v) for v in step.values()) or 1.0
print("# share within the timed step (k_compress<r> + k_psnr only)")
for k, v in sorted(step.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k} | {sum(v) / st:.4f}")
