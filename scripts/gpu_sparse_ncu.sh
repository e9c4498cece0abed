cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for mode in off on; do
OTDR_SPARSE_X=$mode timeout 900 ncu --set full --clock-control none --import-source on -k regex:tstream_kernel -s 1 -c 1 \
  -o gpurun_out/ts_$mode -f python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-ncu > gpurun_out/ncu_ts_$mode.log 2>&1
echo "$mode rc=$?"
done
