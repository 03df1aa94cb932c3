#!/bin/bash
# One GPU call: bench line, ncu launch list of the same command, one --set full capture of K6 and of
# the same-spin kernel. Outputs under gpurun_out/<tag>/ (copy the summaries into profiles/).
#   gpurun --timeout 1500 -- 'bash tools/gpu_profile_round.sh r02_head'
tag=${1:-prof}
out=gpurun_out/$tag
mkdir -p $out
python bench.py --steps 10 --warmup 3 > $out/bench.json 2> $out/bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-tte --no-cpu-baseline > $out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sigma_ab -s 1 -c 1 -o $out/k6 -f \
    python tools/ab_breakdown.py c4 0 > $out/ncu_k6.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sigma_ss -s 2 -c 1 -o $out/ss -f \
    python tools/ab_breakdown.py c4 0 > $out/ncu_ss.log 2>&1
ls -la $out
