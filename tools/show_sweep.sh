for f in "$@"; do echo "== $f"; python -c "
import json,sys
for l in open('$f'):
    try: d=json.loads(l)
    except: print(l.strip()[:200]); continue
    print(d.get('op'),d.get('k'),d.get('us'),d.get('gbs'),d.get('frac'))
"; done
