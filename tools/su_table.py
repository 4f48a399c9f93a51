import collections, json, sys
rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')]
t = collections.defaultdict(dict)
for r in rows:
    t[r['program']][r['tag']] = r['us']
tags = sorted({r['tag'] for r in rows})
print('program'.ljust(14), ' '.join(x.rjust(11) for x in tags))
for p, v in t.items():
    print(p.ljust(14), ' '.join(str(v.get(x, '')).rjust(11) for x in tags))
