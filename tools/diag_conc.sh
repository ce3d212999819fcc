cd $GRAFT_REPO_ROOT
summ() { python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['cap'], d['iter'], [r['timeouts'] for r in d['ranks']])
    elif 'rror' in l: print(l.strip()[:200])" | tr '\n' ' '; echo; }
echo "== P=4 cap 36 PDL off"; PERSEUS_PDL=0 timeout 100 python tools/conc_diag.py 4 36 5 0 2>&1 | summ
echo "== P=2 cap 74 trace PDL off"; PERSEUS_PDL=0 DIAG_TRACE=1 timeout 100 python tools/conc_diag.py 2 74 10 0 2>&1 | summ
echo "== P=3 cap 48 PDL off"; PERSEUS_PDL=0 timeout 100 python tools/conc_diag.py 3 48 5 0 2>&1 | summ
