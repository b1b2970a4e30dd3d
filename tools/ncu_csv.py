"""Summarise an ncu --csv metrics log: one line per launch (time, DRAM bytes, L2 bytes, instructions)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
d = defaultdict(dict)
name = {}
for r in rows[1:]:
    i = int(r[ix["ID"]])
    name[i] = r[ix["Kernel Name"]][:40]
    try:
        d[i][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    except ValueError:
        pass
for i, v in sorted(d.items()):
    g = lambda k, s=1.0: v.get(k, float("nan")) * s
    print(f"{i:3d} {name[i]:40s} t={g('gpu__time_duration.sum', 1e-6):7.3f}ms dram rd={g('dram__bytes_read.sum', 1e-9):6.2f}GB "
          f"wr={g('dram__bytes_write.sum', 1e-9):6.2f}GB L2 rd={g('lts__t_sectors_srcunit_tex_op_read.sum', 32e-9):6.2f}GB "
          f"wr={g('lts__t_sectors_srcunit_tex_op_write.sum', 32e-9):6.2f}GB inst={g('sm__inst_executed.sum', 1e-9):5.2f}G")
