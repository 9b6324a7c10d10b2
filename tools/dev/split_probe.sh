# SwiGLU / down GEMM grid-shape probe: whole tiles vs stream-K with fused fixup
# (SwiGLU), tile-aligned splits vs stream-K ranges (down), at M 64 / 128 / 160.
mkdir -p gpurun_out/sp
for M in 64 128 160; do
  for W in 70 0; do
    for E in 2 0; do
      timeout 300 python tools/profile_kernels.py --only ffn --rows $M --whole $W --even $E \
        --json gpurun_out/sp/M${M}_w${W}_e${E}.json > /dev/null 2>&1
      python -c "import json;d=json.load(open('gpurun_out/sp/M${M}_w${W}_e${E}.json'));print('M$M w$W e$E', *(f\"{k}={v['us']:.1f}\" for k,v in d.items() if 'graph' in k))"
    done
  done
done
