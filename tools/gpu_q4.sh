timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "weight_streaming" 2>&1 | tail -3
for c in 0 1; do echo "cluster $c"; timeout 300 python tools/profile_kernels.py --only ffn --iters 16 --cluster $c 2>&1 | python -c "
import json,sys; t=sys.stdin.read(); d=json.loads(t[t.index(\"{\"):])
print({k: round(v[\"us\"],1) for k,v in d.items() if \"graph\" in k})
"; done
