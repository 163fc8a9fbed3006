"""Instruction mix of every backward-branch loop in a SASS dump (cuobjdump -sass), for
reading kernel inner loops before spending GPU time.  usage: sass_loops.py dump.sass"""
import re
import sys

ins = []
for line in open(sys.argv[1]).read().splitlines():
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s*(.*?);', line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, t) in enumerate(ins):
    m = re.search(r'BRA\s+(?:\S+\s+)?0x([0-9a-f]+)', t)
    if m and int(m.group(1), 16) < a and int(m.group(1), 16) in addr:
        body = ins[addr[int(m.group(1), 16)]:i + 1]
        ops = {}
        for _, tt in body:
            op = (tt.split()[1] if tt.startswith('@') else tt.split()[0]).split('.')[0]
            ops[op] = ops.get(op, 0) + 1
        top = sorted(ops.items(), key=lambda x: -x[1])[:12]
        print(f"{body[0][0]:#06x} -> {a:#06x}  {len(body):4d} instr  " + " ".join(f"{k}:{v}" for k, v in top))
