# small-LP regime: conditional graph vs plain graph (+PDL)
mkdir -p gpurun_out
for v in "HPR_PLAIN=0 HPR_PDL=0" "HPR_PLAIN=0 HPR_PDL=1" "HPR_PLAIN=1 HPR_PDL=0" "HPR_PLAIN=1 HPR_PDL=1"; do
  echo "== $v"; env $v timeout 600 python tools/small_lp_probe.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], d['tol'], d['iterations'], round(d['us_per_it'],2), round(d['create_s'],3), d['status'])"
done
