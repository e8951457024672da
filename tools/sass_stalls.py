"""Sum of the compiler-set stall counts (SASS control bits [105:109)) over one tile body of each
zonal compress kernel: the single-warp issue time of the body if no scoreboard wait occurs.
With W resident warps per SM sub-partition, issue can be saturated only if sum(stall) <= W * body."""
import glob, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
objs = sys.argv[1:] or sorted(glob.glob(os.path.join(ROOT, "build/obj/zonal_part*.o")))
for o in objs:
    sass = subprocess.run(["cuobjdump", "-sass", o], capture_output=True, text=True).stdout
    for blk in sass.split("Function : ")[1:]:
        name = blk.split("\n")[0]
        m = re.search(r"k_compressILi(\d+)E", name)
        if not m or int(m.group(1)) not in (1, 3, 6, 10, 15, 21, 28, 36):
            continue
        lines = blk.split("\n")
        ins = []
        for i, line in enumerate(lines):
            mm = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)[^;]*;\s*/\* (0x[0-9a-f]+) \*/", line)
            if mm:
                hi = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1])
                h = int(hi.group(1), 16) if hi else 0
                ins.append((mm.group(2).split(".")[0], (h >> 41) & 0xF, (h >> 45) & 1))
        body = [i for i, x in enumerate(ins) if x[0] in ("LDS", "FFMA2", "FADD2")]
        waits = [i for i, x in enumerate(ins) if x[0] == "SYNCS" and i > body[0]]
        seg = ins[body[0]:waits[0]] if waits else ins[body[0]:body[-1]]
        st = sum(x[1] for x in seg)
        hist = [sum(1 for x in seg if x[1] == k) for k in range(16)]
        print(f"r={m.group(1):>2} body {len(seg):4d} instr, sum(stall) {st:5d} cycles = {st / len(seg):.2f}/instr, "
              f"stall histogram 1..6: {hist[1:7]}")
