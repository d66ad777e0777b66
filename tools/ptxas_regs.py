"""Registers / spills per kernel from build_ptxas.log: python tools/ptxas_regs.py [substr...]"""
import re, sys
cur = None; info = {}
for line in open('build_ptxas.log'):
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m: cur = m.group(1); info[cur] = {}; continue
    m = re.search(r"Function properties for (\w+)", line)
    if m: cur = m.group(1); info.setdefault(cur, {}); continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur: info[cur]['spill'] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur: info[cur]['regs'] = int(m.group(1))
keys = sys.argv[1:] or ['k_p']
for k, v in info.items():
    if any(s in k for s in keys): print(k[:70], v)
