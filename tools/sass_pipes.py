"""Static per-r pipe estimate of the zonal compress kernels from their SASS (build/obj/zonal_part*.o):
counts ALU-pipe (IADD3/LOP3/PRMT/SHF/ISETP/SEL/LEA/I2FP/PLOP3) and FMA-pipe (FFMA2/FADD2/FMUL2/IMAD/
HADD2/FFMA/FADD) instructions between the first and last LDS/F*2 of the tile body (one ring stage).
B200 issue: 1 warp-instr/clk/SMSP; ALU and FMA pipes 0.5 warp-instr/clk each for these ops
(profiles/r01_pipes_microbench*.txt).  Budget at the measured HBM rate: 729 cycles per 4 KB tile."""
import re, subprocess, sys, glob, os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALU = ("IADD3", "LOP3", "PRMT", "SHF", "ISETP", "SEL", "LEA", "I2FP", "PLOP3", "IADD")
FMA = ("FFMA2", "FADD2", "FMUL2", "IMAD", "HADD2", "FFMA", "FADD", "FMUL", "HFMA2")
FMA1 = ("FHFMA", "FFMA", "FADD", "FMUL")  # full-rate FMA-pipe ops: 1 cycle (the others 2)
objs = sys.argv[1:] or sorted(glob.glob(os.path.join(ROOT, "build/obj/zonal_part*.o")))
res = {}
for o in objs:
    sass = subprocess.run(["cuobjdump", "-sass", o], capture_output=True, text=True).stdout
    for blk in sass.split("Function : ")[1:]:
        name = blk.split("\n")[0]
        m = re.search(r"k_compressILi(\d+)E.*?ELb([01])E", name)
        if not m:
            continue
        ops = []
        for line in blk.split("\n"):
            mm = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
            if mm:
                ops.append(mm.group(2).split(".")[0])
        body = [i for i, op in enumerate(ops) if op in ("LDS", "FFMA2", "FADD2")]
        # two ring stages are unrolled: take the first body (up to the second SYNCS wait)
        waits = [i for i, op in enumerate(ops) if op == "SYNCS" and i > body[0]]
        seg = ops[body[0]:waits[0]] if waits else ops[body[0]:body[-1]]
        alu = sum(op in ALU for op in seg)
        fma = sum(op in FMA for op in seg) + sum(op in FMA1 for op in seg)
        fcyc = 2 * sum(op in FMA and op not in FMA1 for op in seg) + sum(op in FMA1 for op in seg)
        res[int(m.group(1))] = (len(seg), alu, fma, m.group(2), fcyc)
print(" r  resid  body-instr  ALU  FMA   pipe-cycles  bound(frac of 729)")
for r in sorted(res):
    n, a, f, rs, fcyc = res[r]
    cyc = max(n, 2 * a, fcyc)
    print(f"{r:2d}  {rs}      {n:5d}     {a:4d} {f:4d}   {cyc:5d}        {729 / cyc:.2f}")
