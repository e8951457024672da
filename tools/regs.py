"""Print registers / spill bytes of the zonal compress instantiations from the build logs."""
import re, sys, os
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for part in range(4):
    s = open(os.path.join(root, f'build/obj/zonal_part{part}.o.log')).read()
    out = []
    for e in re.split(r"ptxas info    : Compiling entry function '", s)[1:]:
        name = e.split("'")[0]
        r = re.search(r'ILi(\d+)E', name).group(1)
        regs = re.search(r'Used (\d+) registers', e).group(1)
        sp = re.search(r'(\d+) bytes spill stores', e).group(1)
        out.append(f"{r}:{regs}/{sp}")
    print(' '.join(sorted(out, key=lambda x: int(x.split(':')[0]))))
