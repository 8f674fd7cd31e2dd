"""Print the headline numbers and per-kernel table of bench JSON lines (profiles helper)."""
import json, sys
for f in sys.argv[1:]:
    lines = [x for x in open(f) if x.startswith('{')]
    if not lines:
        print(f, 'no JSON line'); continue
    d = json.loads(lines[-1])
    print(f, 'ms/step', round(d['ms_per_step'], 3), 'value', round(d['value']), d.get('clocks'))
    for k, v in d.get('kernels', {}).items():
        print('   ', k, round(v['ms_per_step'], 3), {kk: round(vv, 3) for kk, vv in v.items() if 'frac' in kk})
    b = d.get('baselines') or {}
    if b: print('    baselines', {k: (round(v, 2) if isinstance(v, float) else v) for k, v in b.items()})
