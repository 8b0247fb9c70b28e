for sz in "128 128 80" "256 256 80" "512 512 80" "1024 1024 80"; do
echo "== $sz"
timeout 600 python tools/reduce_variants.py $sz 0,20 2>&1 | python -c "
import sys,json
rows={}
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); rows.setdefault(d['name'],[]).append(f\"{d['variant']}:{d['us']:.1f}/{d['frac']:.2f}{'' if d.get('bitwise',True) else 'MISMATCH'}\")
for k,v in rows.items(): print(k,' '.join(v))
"
done
