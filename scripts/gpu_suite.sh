cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python benchmarks/configs.py cfg1 > gpurun_out/cfg1.log 2>&1; cut -c1-200 gpurun_out/cfg1.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
