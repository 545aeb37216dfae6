"""ptxas / SASS summary of the hot kernels of libp2m_cuda.so: registers, spills (ptxas -v log written by
the Makefile), and SASS mnemonic counts (cuobjdump): packed f32x2 math, fp64 math, local-memory
traffic, shuffles / REDUX, shared atomics, async copies.  usage: python scripts/sass_summary.py > OUT"""
import collections, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2605_00429_b200", "lib", "libp2m_cuda.so")
log = open(os.path.join(ROOT, "paper_2605_00429_b200", "lib", "ptxas.log")).read()
hot = ("k_scan_warpq", "k_scan_tiles", "k_scan_small", "k_descend", "k_query", "k_morton", "k_table_miss")
info = {}
for m in re.finditer(r"Function properties for (\S+)\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\nptxas info\s+: Used (\d+) registers[^\n]*?(?:, (\d+) bytes smem)?\n", log):
    info[m.group(1)] = dict(stack=int(m.group(2)), st=int(m.group(3)), ld=int(m.group(4)), regs=int(m.group(5)), smem=int(m.group(6) or 0))
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, counts = None, collections.defaultdict(collections.Counter)
for line in sass.split("\n"):
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,6}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        counts[cur][m.group(1)] += 1
groups = [("f32x2 (FADD2/FMUL2/FFMA2)", ("FADD2", "FMUL2", "FFMA2")), ("fp64 (DADD/DMUL/DFMA/DSETP)", ("DADD", "DMUL", "DFMA", "DSETP")),
          ("LDL", ("LDL",)), ("STL", ("STL",)), ("LDS", ("LDS",)), ("STS", ("STS",)), ("LDG", ("LDG",)), ("STG", ("STG",)),
          ("SHFL", ("SHFL",)), ("REDUX", ("REDUX",)), ("VOTE", ("VOTE",)), ("ATOMS", ("ATOMS",)), ("LDGSTS (cp.async)", ("LDGSTS",)),
          ("UBLKCP/UTMALDG (bulk/TMA)", ("UBLKCP", "UTMALDG")), ("BAR", ("BAR",))]
print("kernel | regs | stack B | spill st/ld B | smem B | SASS instrs | " + " | ".join(g[0] for g in groups))
for fn in sorted(counts):
    if not any(h in fn for h in hot) or "cub" in fn:
        continue
    i = info.get(fn, {})
    c = counts[fn]
    short = re.sub(r"^_ZN3p2m3dev\d+_GLOBAL__N__\w+?_cu_\w{8}", "", fn)
    short = next((h for h in hot if h in fn), short) + ("<counters>" if "ILb1E" in fn else "<>" if "ILb0E" in fn else "")
    print(f"{short} | {i.get('regs', '?')} | {i.get('stack', '?')} | {i.get('st', '?')}/{i.get('ld', '?')} | {i.get('smem', '?')} | {sum(c.values())} | "
          + " | ".join(str(sum(c[k] for k in g[1])) for g in groups))
