timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python tools/profile_kernels.py --only ffn --iters 24 2>&1 | python -c "
import json,sys; t=sys.stdin.read(); d=json.loads(t[t.index(\"{\"):])
print({k: round(v[\"us\"],1) for k,v in d.items()})
"
