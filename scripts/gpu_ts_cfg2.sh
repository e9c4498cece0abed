cd $GRAFT_REPO_ROOT
for c in 0 3; do
  echo "== ts_cfg $c"
  OTDR_TS_CFG=$c timeout 600 python benchmarks/configs.py cfg2 cfg4 2>&1 | cut -c1-400
  OTDR_TS_CFG=$c timeout 600 python benchmarks/shard_projection.py 1 4 8 2>&1 | cut -c1-300
done
