cd $GRAFT_REPO_ROOT
for v in "" "OTDR_GL_PIPE_NT=256" "OTDR_GL_PIPE_W=64" "OTDR_GL_PIPE_NT=256 OTDR_GL_PIPE_G=16" ""; do
  echo "== $v"; env $v timeout 600 python benchmarks/configs.py cfg3 2>&1 | cut -c1-330
done
if [ -n "$TESTS" ]; then OTDR_GL_PIPE_NT=256 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$TESTS" 2>&1 | tail -3; fi
