"""Per-kernel summary of an ncu --csv metrics log (tools/edt_profile.sh):
mean duration, warp instructions, threads/inst and DRAM bytes per launch."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
per = collections.defaultdict(dict)
for r in rows[1:]:
    try:
        v = float(r[ix["Metric Value"]].replace(",", ""))
    except ValueError:
        continue
    per[(int(r[ix["ID"]]), r[ix["Kernel Name"]])][r[ix["Metric Name"]]] = v
agg = collections.defaultdict(list)
order = []
for (i, name), m in sorted(per.items()):
    short = name.split("(")[0].replace("void vx::<unnamed>::", "").replace("vx::<unnamed>::", "")
    if short not in agg:
        order.append(short)
    agg[short].append(m)
print(f"{'kernel':60s} {'n':>3s} {'us':>9s} {'Mwinst':>8s} {'thr/i':>6s} {'DRAM MB':>9s}")
for k in order:
    ms = agg[k]
    f = lambda key: sum(m.get(key, 0.0) for m in ms) / len(ms)  # noqa: E731
    print(f"{k[:60]:60s} {len(ms):3d} {f('gpu__time_duration.sum')/1e3:9.1f} "
          f"{f('smsp__inst_executed.sum')/1e6:8.1f} {f('smsp__thread_inst_executed_per_inst_executed.ratio'):6.1f} "
          f"{(f('dram__bytes_read.sum') + f('dram__bytes_write.sum'))/1e6:9.1f}")
