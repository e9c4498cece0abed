cd $GRAFT_REPO_ROOT
echo "== wide (default)"; timeout 300 python benchmarks/configs.py cfg1 2>&1 | cut -c1-330
echo "== f32 tiles"; OTDR_RESIDENT_TILES=f32 timeout 300 python benchmarks/configs.py cfg1 2>&1 | cut -c1-330
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size_parity.py tests/test_optimality_oracles.py -m gpu -x -q -k "resident or cfg1 or first_step or headline_k or fp32 or oracle" 2>&1 | tail -4
