import collections, json, sys
rows = [json.loads(l) for l in open(sys.argv[1])]
t = collections.defaultdict(dict)
for r in rows:
    t[(r["cfg"], r.get("op", "spmm"), r["tag"])][r["k"]] = r["gbs"]
for key, v in sorted(t.items()):
    print(key, v)
