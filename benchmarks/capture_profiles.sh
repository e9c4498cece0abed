#!/bin/bash
# Round profile capture on one B200 (run under gpurun from the repo root).
# Writes gpurun_out/: bench.log (the driver line), launches.csv (ncu launch
# list of the driver's exact bench command, --steps 20 --warmup 5),
# stream.ncu-rep (--set full of the timed streaming-kernel launch of that
# command: 20 iterations after the 5 warm-up ones), sweep.ncu-rep (graph-path
# sweep kernel), gl.ncu-rep / glstream.ncu-rep (cfg3 group-lasso sweep).
# gpurun copies back at most 64 MiB, so run it as two calls:
#   capture_profiles.sh a   (bench, launch list, stream + sweep reports)
#   capture_profiles.sh b   (group-lasso reports, configs, GPU tests)
set -u
mkdir -p gpurun_out
part=${1:-a}
if [ "$part" = a ]; then
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-ncu \
  > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 1 -c 1 \
  -o gpurun_out/stream -f python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-ncu > gpurun_out/ncu_stream.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 \
  -o gpurun_out/sweep -f python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-ncu > gpurun_out/ncu_sweep.log 2>&1
fi
if [ "$part" = b ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gl_pipe -s 3 -c 1 \
  -o gpurun_out/gl -f python benchmarks/variants.py cfg3 > gpurun_out/ncu_gl.log 2>&1

timeout 600 ncu --set full --clock-control none --import-source on -k regex:gl_stream -s 1 -c 1 \
  -o gpurun_out/glstream -f python benchmarks/gl_step.py > gpurun_out/ncu_glstream.log 2>&1
timeout 600 python benchmarks/configs.py cfg1 cfg2 cfg3 cfg4 cfg5 > gpurun_out/configs.log 2>&1

fi
echo all_done
