# GPU test pass: full -m gpu suite + smoke; logs under gpurun_out/.
mkdir -p gpurun_out
timeout ${T:-2400} python -m pytest tests -m gpu -q ${ARGS:--x} > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/gpu_tests.log
