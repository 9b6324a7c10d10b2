#!/bin/bash
# compute-sanitizer passes over the kernel parity tests: memcheck
# (out-of-bounds / misaligned global + shared accesses), racecheck (shared
# memory hazards), synccheck (barrier misuse). Logs + summaries under
# gpurun_out/sanitize_*.log. Usage (on the GPU box): bash tools/sanitize.sh
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL_ALL="test_gemm_weight_streaming or test_expert_ffn or test_permute or test_combine or test_decode_attention_split_kv or test_gemm_split_k or test_gemm_residual or test_gate_topk or test_coact or test_prefill_attention_window or test_rope or test_q4 or test_gemm_store or test_gemm_persistent"
SEL_SMALL="test_gemm_weight_streaming or test_expert_ffn or test_permute or test_combine or test_decode_attention_split_kv or test_gemm_split_k or test_prefill_attention_window"
run() {  # tool, selection, timeout
    timeout "$3" $CS --tool "$1" --target-processes all --print-limit 20 \
        python -m pytest tests/test_kernels_gpu.py -m gpu -q -p no:cacheprovider -k "$2" \
        > "gpurun_out/sanitize_$1.log" 2>&1
    echo "$1 rc=$? $(grep -h 'ERROR SUMMARY' gpurun_out/sanitize_$1.log | sort | uniq -c | tr '\n' ';') $(tail -1 gpurun_out/sanitize_$1.log)"
}
run memcheck "$SEL_ALL" ${T_MEM:-1500}
run synccheck "$SEL_SMALL" ${T_SYNC:-900}
run racecheck "$SEL_SMALL" ${T_RACE:-1500}
