"""SASS opcode mix (executed warp instructions) of one kernel in an ncu report:
python tools/ncu_sass_mix.py rep.ncu-rep <kernel-regex> [top]"""
import collections, csv, io, subprocess, sys

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass',
                      '--kernel-id', f'::regex:{rx}:1'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si, ei = h.index('Source'), h.index('Instructions Executed')
wi = h.index('Warp Stall Sampling (All Samples)')
ops, stall, tot, st = collections.Counter(), collections.Counter(), 0, 0
for r in rows[2:]:
    try:
        e = int(r[ei])
    except (ValueError, IndexError):
        continue
    toks = r[si].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith('@') else toks[0]
    op = op.split('.')[0]
    ops[op] += e
    w = int(r[wi] or 0)
    stall[op] += w
    tot += e
    st += w
print(f'{rx}: {tot} warp instructions, {st} stall samples')
for op, c in ops.most_common(top):
    print(f'  {op:10s} {c:11d} {100 * c / tot:5.1f}%   stall {100 * stall[op] / max(st, 1):5.1f}%')
