timeout 900 python -m pytest tests -m gpu -q -x -k "mixtral_shape or expert_ffn" 2>&1 | tail -4
