"""Map local-memory (STL/LDL) instructions of a kernel to source lines, split
by warp-role region (setmaxnreg dealloc = producer side, alloc = consumers).
usage: python tools/spills.py <cubin> <function-substring> [top]"""
import collections, re, subprocess, sys

sass = subprocess.run(["nvdisasm", "-g", "-c", sys.argv[1]], capture_output=True, text=True).stdout
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cur, fn, region, cnt = None, None, "pre", collections.Counter()
for line in sass.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m:
        fn, region = m.group(1), "pre"
    m = re.search(r'//## File ".*/(\S+)", line (\d+)', line)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    if not fn or want not in fn:
        continue
    if "USETMAXREG.DEALLOC" in line:
        region = "prod"
    if "USETMAXREG.TRY_ALLOC" in line:
        region = "cons"
    if re.search(r"\b(STL|LDL)", line):
        cnt[(region, cur, "STL" if "STL" in line else "LDL")] += 1
tot = collections.Counter()
for (r, _, _), v in cnt.items():
    tot[r] += v
print("local-memory instructions per region:", dict(tot))
for k, v in sorted(cnt.items(), key=lambda x: -x[1])[:top]:
    print(f"{v:4d} {k[0]:5s} {k[2]} {k[1]}")
