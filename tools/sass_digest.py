"""SASS digest of libpswe.so: per kernel, the instruction mix that proves the FP64 tensor path
(DMMA.8x8x4 - tcgen05 has no f64 kind, so mma.sync f64 is Blackwell's FP64 tensor instruction),
the bulk copies (UBLKCP = cp.async.bulk, TMA engine) and mbarrier traffic (SYNCS), and the
register / shared-memory footprint from cuobjdump -res-usage.
Usage: python tools/sass_digest.py [lib.so] > profiles/r02_sass_digest.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1904_05988_b200/libpswe.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
OPS = ["DMMA", "UBLKCP", "SYNCS", "LDGSTS", "LDS", "STS", "LDG", "STG", "DFMA", "DADD", "DMUL", "BAR", "SHFL"]
counts = collections.OrderedDict()
name = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        counts[name] = collections.Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.x]+)?", line)
    if name and m:
        op = m.group(2)
        for o in OPS:
            if op == o or (o == "SYNCS" and op.startswith("SYNCS")):
                counts[name][o] += 1
usage = {}
for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:(\d+)", res):
    usage[m.group(1)] = (int(m.group(2)), int(m.group(3)), int(m.group(4)))


def short(n):
    d = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"pswe::\(anonymous namespace\)::", "", d)
    return re.sub(r"\(.*", "", d)


print(f"# SASS digest of {lib} (cuobjdump -sass / -res-usage); kernels with DMMA, bulk copies or mbarriers first")
print(f"{'kernel':58s} {'REG':>4s} {'SMEM':>6s} " + " ".join(f"{o:>6s}" for o in OPS))
rows = sorted(counts.items(), key=lambda kv: -(kv[1]["DMMA"] * 10 + kv[1]["UBLKCP"] + kv[1]["SYNCS"]))
for n, c in rows:
    u = usage.get(n, (0, 0, 0))
    print(f"{short(n)[:58]:58s} {u[0]:4d} {u[2]:6d} " + " ".join(f"{c[o]:6d}" for o in OPS))
tot = collections.Counter()
for c in counts.values():
    tot.update(c)
print(f"# totals over {len(counts)} kernels: " + ", ".join(f"{o} {tot[o]}" for o in OPS))
