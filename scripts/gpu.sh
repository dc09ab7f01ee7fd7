#!/usr/bin/env bash
# One parameterised runner for gpurun calls (replaces the round-1 one-off gpu_*.sh scripts).
#   gpurun --timeout S -- 'bash scripts/gpu.sh <task> [args...]'
# Tasks (each writes its logs under gpurun_out/ and prints a one-line summary per run):
#   test [pytest -k expr]      pytest -m gpu (+ smoke)
#   bench [bench.py args]      one bench.py line
#   configs                    every BASELINE config once at N=1 (+ the extra precision rows)
#   launches [bench.py args]   ncu launch list (gpu__time_duration) of a bench command, after it ran clean
#   ncu <regex> <name> [args]  one ncu --set full capture of the first launch matching <regex>
#   ab VAR "v1 v2" [args]      A/B of env-selected variants, alternated twice
#   multirank                  bench.py's multi-rank path on one GPU (gloo ranks on device 0)
#   sweep [motions...]         c2 network in bf16 over motion counts
#   latency                    per-call predict_min_distance latency from C++ (scripts/latency_cpp.cpp)
#   rzsweep [c...]             fp32_split error per calibration seed for truncation compensations c
set -u
mkdir -p gpurun_out
task=${1:-test}; shift || true
line() { tail -1 "$1" | python scripts/benchline.py "$2"; }
case "$task" in
  test)
    nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
    if [ $# -gt 0 ]; then K=(-k "$*"); else K=(); fi
    timeout 2400 python -m pytest tests -m gpu -q -x "${K[@]}" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
    tail -5 gpurun_out/pytest_gpu.log ;;
  bench)
    timeout 1800 python bench.py "$@" > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
    line gpurun_out/bench.log "bench $*" ;;
  configs)
    for a in "--config c1" "--config c2" "--config c3" "--config c4" "--config c5single" \
             "--config c1 --precision fp32_split" "--config c2 --precision fp32_split" \
             "--config c1 --precision bf16" "--config c2 --precision bf16" "--config paper" \
             "--config c3 --precision fp32_split" "--config c4 --precision fp32_split" "--config c3 --precision fp32" \
             "--config c3 --precision fp16" "--config c4 --precision fp16" "--config c2 --precision fp16" \
             "--config c1 --precision fp16" "--config paper --precision fp16"; do
      n=$(echo "$a" | tr -d ' -'); timeout 900 python bench.py $a --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$n.log 2>&1
      line gpurun_out/cfg_$n.log "$a"
    done ;;
  launches)
    C="python bench.py $* --no-cpu-baseline --no-e2e --no-parity"
    timeout 1800 $C > gpurun_out/launch_plain.log 2>&1 && \
    timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $C \
      > gpurun_out/launch_ncu.log 2>&1; echo "launches rc=$?" ;;
  ncu)
    re=$1; name=$2; shift 2
    C="python bench.py $* --no-cpu-baseline --no-e2e --no-parity"
    timeout 1800 $C > gpurun_out/ncu_plain_$name.log 2>&1 && \
    timeout 1800 ncu --set full --clock-control none --import-source on -k regex:$re -s 1 -c 1 -o gpurun_out/$name $C \
      > gpurun_out/ncu_$name.log 2>&1; echo "ncu $name rc=$?" ;;
  ab)
    var=$1; vals=$2; shift 2; i=0
    for rep in 1 2; do for v in $vals; do i=$((i+1))
      env $var=$v timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-parity "$@" \
        > gpurun_out/ab_$i.log 2>&1; line gpurun_out/ab_$i.log "$var=$v $*"
    done; done ;;
  multirank)
    export SVN_BENCH_BACKEND=gloo SVN_BENCH_DEVICE=0
    timeout 900 python bench.py --gpus 2 --config c3 --motions 64 --steps 3 --warmup 3 --no-cpu-baseline \
      > gpurun_out/mr_motion.log 2>&1; line gpurun_out/mr_motion.log "2 ranks motion"
    timeout 900 python bench.py --gpus 2 --config c5single --points 2000000 --steps 3 --warmup 3 --no-cpu-baseline \
      > gpurun_out/mr_point.log 2>&1; line gpurun_out/mr_point.log "2 ranks point"
    unset SVN_BENCH_BACKEND SVN_BENCH_DEVICE
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
      --master-port 29536 bench.py --gpus 1 --config c3 --steps 3 --warmup 3 > gpurun_out/mr_nccl1.log 2>&1
    line gpurun_out/mr_nccl1.log "torchrun nccl N=1" ;;
  sweep)
    for m in ${@:-16 32 64 128 256 512 1024}; do
      timeout 600 python bench.py --config c2 --precision bf16 --motions $m --steps 4 --warmup 3 --no-cpu-baseline \
        --no-e2e --no-parity > gpurun_out/sw_$m.log 2>&1; line gpurun_out/sw_$m.log "c2 bf16 M=$m"
    done ;;
  latency)
    g++ -std=c++17 -O2 -Iinclude scripts/latency_cpp.cpp -Lpaper_2402_15281_b200/_lib -lsweptnet_b200 \
      -Wl,-rpath,$PWD/paper_2402_15281_b200/_lib -o gpurun_out/latency_cpp && \
    for v in ${LAT_GRAPH:-1}; do echo "SVN_GRAPH=$v"; SVN_GRAPH=$v timeout 300 gpurun_out/latency_cpp; done 2>&1 | tee gpurun_out/latency.log ;;
  rzsweep)
    for c in ${@:-0 0.25}; do SVN_SPLIT_RZ=$c timeout 900 python scripts/split_rz_sweep.py; done 2>&1 | tee gpurun_out/rzsweep.log ;;
  *) echo "unknown task $task"; exit 2 ;;
esac
