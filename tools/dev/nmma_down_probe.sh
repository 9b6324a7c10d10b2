# Down-projection GEMM with one vs two 128-row weight sub-tiles per activation
# tile (activation re-reads from L2 halve with 2), at M 64 / 128 / 160.
mkdir -p gpurun_out/nd
for M in 64 128 160; do
  for N in 1 2; do
    timeout 300 python tools/profile_kernels.py --only ffn --rows $M --nmma $N \
      --json gpurun_out/nd/M${M}_n${N}.json > gpurun_out/nd/M${M}_n${N}.log 2>&1
    python -c "import json;d=json.load(open('gpurun_out/nd/M${M}_n${N}.json'));print('M$M nmma$N', *(f\"{k}={v['us']:.1f}\" for k,v in d.items() if 'graph' in k))"
  done
done
