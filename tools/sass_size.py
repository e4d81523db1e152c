"""SASS bytes per source function of a kernel (development aid): instruction
cache pressure check. usage: sass_size.py file.cu [nvcc flags]"""
import collections, re, subprocess, sys
src_path = sys.argv[1]
subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-cubin", "-o", "/tmp/sz.cubin", src_path] + sys.argv[2:], check=True)
dis = subprocess.run(["/usr/local/cuda/bin/nvdisasm", "-g", "-c", "/tmp/sz.cubin"], capture_output=True, text=True).stdout
cur = None; cnt = collections.Counter(); kern = None; kcnt = collections.Counter()
for line in dis.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m: kern = m.group(1)
    m = re.search(r'//## File "(.*)", line (\d+)', line)
    if m: cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        if cur: cnt[cur] += 1
        if kern: kcnt[kern] += 1
src = open(src_path).read().split("\n")
funcs = [(i, m.group(1)) for i, l in enumerate(src, 1) for m in [re.match(r"^(?:__device__|__global__)[^(]*?(\w+)\(", l)] if m]
def fn(line):
    name = "?"
    for i, n in funcs:
        if i <= line: name = n
    return name
agg = collections.Counter()
base = src_path.split("/")[-1]
for (f, l), c in cnt.items():
    agg[fn(l) if f == base else f] += c
for k, v in kcnt.most_common(6): print(f"{v * 16:8d} bytes  kernel {k[:80]}")
for k, v in agg.most_common(15): print(f"{v * 16:8d} bytes  {k}")
