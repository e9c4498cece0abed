cd $GRAFT_REPO_ROOT
bash benchmarks/capture_profiles.sh a; echo "capture a rc=$?"
timeout 600 python benchmarks/shard_projection.py > gpurun_out/shard_projection.jsonl 2>&1; echo "proj rc=$?"
OTDRB_M=40000 timeout 900 python benchmarks/shard_projection.py > gpurun_out/shard_projection_40000.jsonl 2>&1; echo "proj40k rc=$?"
timeout 900 python benchmarks/e2e_breakdown.py > gpurun_out/e2e_breakdown.jsonl 2>&1; echo "e2e rc=$?"
