cd $GRAFT_REPO_ROOT
b() { timeout 150 python bench.py --steps 20 --warmup 5 --no-cpu --no-ncu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],1), d['time_to_tol']['iterations'], round(d['time_to_tol']['device_s'],4))"; }
for c in ${CFGS:-0 3 0 3}; do OTDR_TS_CFG=$c b cfg$c; done
if [ -n "$TESTS" ]; then timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$TESTS" 2>&1 | tail -2; fi
if [ -n "$CONFIGS" ]; then for c in 0 3; do OTDR_TS_CFG=$c timeout 600 python benchmarks/configs.py cfg2 2>&1 | cut -c1-200; OTDR_TS_CFG=$c timeout 600 python benchmarks/shard_projection.py 8 2>&1 | cut -c1-300; done; fi
