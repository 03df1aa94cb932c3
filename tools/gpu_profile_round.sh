#!/bin/bash
# One GPU call: bench line, ncu launch list of the same command, one --set full capture of K6 and of
# the same-spin kernel, reduced to text on the box (the .ncu-rep files are too large to bring back).
#   gpurun --timeout 1800 -- 'bash tools/gpu_profile_round.sh r02_final'
tag=${1:-prof}
out=gpurun_out/$tag
mkdir -p $out
python bench.py --steps 10 --warmup 3 > $out/bench.json 2> $out/bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-tte --no-cpu-baseline > $out/ncu_launch.log 2>&1
python tools/launches.py $out/launches.csv > $out/launches.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sigma_ab -s 1 -c 1 -o /tmp/k6 -f \
    python tools/ab_breakdown.py c4 0 > $out/ncu_k6.log 2>&1
python tools/ncu_summary.py /tmp/k6.ncu-rep > $out/ncu_full_c4_k6_summary.txt 2>&1
python tools/ncu_stalls.py /tmp/k6.ncu-rep 30 > $out/ncu_full_c4_k6_stalls.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sigma_ss -s 2 -c 1 -o /tmp/ss -f \
    python tools/ab_breakdown.py c4 0 > $out/ncu_ss.log 2>&1
python tools/ncu_summary.py /tmp/ss.ncu-rep > $out/ncu_full_c4_ss_summary.txt 2>&1
python tools/ncu_stalls.py /tmp/ss.ncu-rep 30 > $out/ncu_full_c4_ss_stalls.txt 2>&1
ls -la $out
