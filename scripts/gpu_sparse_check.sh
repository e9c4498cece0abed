cd $GRAFT_REPO_ROOT
b() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-ncu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],1), d['time_to_tol']['iterations'], round(d['time_to_tol']['device_s'],4))"; }
OTDR_SPARSE_X=off b off
b on96
OTDR_TS_DENSE=32 b on32
OTDR_TS_DENSE=256 b on256
OTDR_TS_DENSE=600 b on600
OTDR_COMPRESS=off b on_nocomp
OTDR_COMPRESS=off OTDR_TS_DENSE=600 b on600_nocomp
