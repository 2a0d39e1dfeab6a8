"""Opcode histogram of every backward-branch loop in a cuobjdump -sass listing."""
import collections
import re
import sys

ins = []
for l in open(sys.argv[1]):
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, t) in enumerate(ins):
    mm = re.search(r"BRA.*?0x([0-9a-f]+)", t)
    if mm:
        tgt = int(mm.group(1), 16)
        if tgt < a and tgt in addr:
            body = ins[addr[tgt]:i + 1]
            c = collections.Counter((x.split()[1] if x.startswith("@") else x.split()[0]) for _, x in body)
            print(hex(tgt), hex(a), len(body), dict(c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 14)))
