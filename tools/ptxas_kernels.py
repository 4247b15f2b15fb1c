"""Registers / spills / stack per kernel from the build's ptxas log.
    python tools/ptxas_kernels.py [substring ...]"""
import re
import subprocess
import sys

t = open('paper_2403_07221_b200/csrc/build/ptxas.log').read()
blocks = re.split(r"ptxas info\s+: Compiling entry function '", t)
for b in blocks[1:]:
    name = b.split("'")[0]
    dn = subprocess.run(['c++filt', name], capture_output=True, text=True).stdout.strip()
    if sys.argv[1:] and not any(s in dn for s in sys.argv[1:]):
        continue
    m = re.search(r"Used (\d+) registers", b)
    sp = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", b)
    st = re.search(r"(\d+) bytes stack frame", b)
    print(dn[:120], '| regs', m.group(1) if m else '?', '| spill', sp.group(1) + '/' + sp.group(2) if sp else '?',
          '| stack', st.group(1) if st else '?')
