#!/usr/bin/env bash
# tools/gpu.sh -- the measurement recipes run on the GPU box through gpurun
# (replaces round 1's one-off tools/run_*.sh).  Outputs land in gpurun_out/.
#
#   gpurun [--gpus N] -- 'bash tools/gpu.sh <recipe> [args]'
#
# recipes
#   tests [N]            pytest -m gpu on this box (N GPUs visible: the multi-GPU
#                        parity of tests/test_gpu_multi.py runs at every n <= N)
#   bench N CFG [extra]  bench.py at N GPUs (torchrun for N > 1), config CFG
#   table N CFGS...      bench.py --no-e2e for each config at N GPUs
#   scale [N]            the default bench (C2) at 1, 2, ... N GPUs + reference arm
#   timeline N CFG       per-CTA start / end spread of the cast launch (tools/timeline.py)
#   launches CFG         ncu launch list (gpu__time_duration, --clock-control none), 1 GPU
#   ncufull CFG KERNEL   ncu --set full of one kernel (regex), 1 GPU, 1 launch
#   final1               end-of-round evidence on 1 GPU: tests + smoke, the default bench
#                        line, the 1-GPU table, the C2 launch list and ncu capture
#   final4               end-of-round evidence on 4 GPUs: multi-GPU parity (2 and 4), the
#                        4-GPU table incl. C9 three ways, the default bench at 1, 2, 4
#   nvlink N CFG         ncu NVLink + DRAM counters, one process driving N GPUs (NVFP4: the
#                        supplied-amax one-pass sync -- the two-pass handshake would deadlock
#                        under ncu's serialised launches)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=$((29500 + RANDOM % 400))
run_bench() {  # N CFG extra...
    local n=$1 cfg=$2; shift 2
    port=$((port + 1))
    if [ "$n" = 1 ]; then
        timeout 900 python bench.py --config "$cfg" "$@"
    else
        timeout 900 $R --nproc-per-node "$n" --master-port $port bench.py --gpus "$n" --config "$cfg" "$@"
    fi
}
recipe=${1:-tests}; shift || true
case "$recipe" in
tests)
    python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
    timeout 3000 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/pytest_gpu.log 2>&1
    echo "pytest rc=$? ($(git rev-parse --short HEAD 2>/dev/null || echo snapshot))" >> gpurun_out/pytest_gpu.log
    tail -5 gpurun_out/pytest_gpu.log ;;
bench)
    n=$1; cfg=$2; shift 2
    run_bench "$n" "$cfg" "$@" > "gpurun_out/bench_${cfg}_n${n}.json" 2> "gpurun_out/bench_${cfg}_n${n}.err"
    tail -c 600 "gpurun_out/bench_${cfg}_n${n}.json" ;;
table)
    n=$1; shift
    for cfg in "$@"; do
        run_bench "$n" "$cfg" --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
            > "gpurun_out/table_${cfg}_n${n}.json" 2> "gpurun_out/table_${cfg}_n${n}.err"
        python - "$cfg" "$n" <<'EOF'
import json, sys
cfg, n = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/table_{cfg}_n{n}.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(cfg, n, d["value"], r["bound"], r["achieved"], r["frac"], r["t_lb_ms"],
          d.get("nvfp4_supplied_amax", {}).get("value"))
except Exception as e:
    print(cfg, n, "FAILED", e)
EOF
    done ;;
scale)
    top=${1:-4}
    timeout 900 python bench.py > gpurun_out/scale_n1.json 2> gpurun_out/scale_n1.err
    for n in 2 4 8; do
        [ "$n" -le "$top" ] || break
        port=$((port + 1))
        timeout 900 $R --nproc-per-node $n --master-port $port bench.py --gpus $n > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err
    done
    timeout 900 python bench.py --impl reference > gpurun_out/scale_ref_n1.json 2> gpurun_out/scale_ref_n1.err ;;
timeline)
    n=$1; cfg=$2; port=$((port + 1))
    timeout 600 $R --nproc-per-node "$n" --master-port $port tools/timeline.py --gpus "$n" --config "$cfg" \
        > "gpurun_out/timeline_${cfg}_n${n}.jsonl" 2> "gpurun_out/timeline_${cfg}_n${n}.err" ;;
launches)
    cfg=$1
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file "gpurun_out/launches_${cfg}.csv" python bench.py --config "$cfg" --steps 2 --warmup 3 \
        --no-e2e --no-cpu-baseline > "gpurun_out/launches_${cfg}.log" 2>&1 ;;
ncufull)
    cfg=$1; k=$2
    timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$k" -c 1 \
        -o "gpurun_out/ncu_${cfg}_${k}" python bench.py --config "$cfg" --steps 1 --warmup 3 --no-e2e \
        --no-cpu-baseline --no-nv-supplied > "gpurun_out/ncufull_${cfg}.log" 2>&1 ;;
nvlink)
    n=$1; cfg=$2
    timeout ${NVL_TIMEOUT:-600} ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none -k regex:llrl_k_cast --csv --log-file "gpurun_out/nvlink_${cfg}_n${n}.csv" \
        python tools/nvlink_1proc.py "$cfg" "$n" >"gpurun_out/nvlink_${cfg}_n${n}.log" 2>&1 ;;
final1)
    rev=$(cat .git_rev 2>/dev/null || echo snapshot)
    bash "$0" tests
    sed -i "s/(snapshot)/($rev)/" gpurun_out/pytest_gpu.log
    timeout 900 python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err
    bash "$0" table 1 c1 c2 c3 c4 c7 c10 c11 c12 > gpurun_out/final_table_n1.txt 2>&1
    bash "$0" launches c2
    bash "$0" ncufull c2 llrl_k_cast_tma
    ncu -i gpurun_out/ncu_c2_llrl_k_cast_tma.ncu-rep --page raw --csv > gpurun_out/ncu_c2_raw.csv 2>/dev/null
    timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref_n1.json 2> gpurun_out/final_ref_n1.err
    echo "final1 done ($rev)" ;;
final4)
    rev=$(cat .git_rev 2>/dev/null || echo snapshot)
    timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -rs > gpurun_out/pytest_multi.log 2>&1
    echo "pytest rc=$? ($rev)" >> gpurun_out/pytest_multi.log
    timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "graph_replay or long_items or item_order" \
        >> gpurun_out/pytest_multi.log 2>&1
    echo "pytest (1-GPU subset) rc=$? ($rev)" >> gpurun_out/pytest_multi.log
    bash "$0" table 4 c2 c3 c4 c5 c6 c7 c8 c10 c11 c12 > gpurun_out/final_table_n4.txt 2>&1
    for extra in "--multicast" "--step-sync" "--replicate nccl --step-sync"; do
        port=$((port + 1))
        tag=$(echo $extra | tr -d ' -')
        timeout 600 $R --nproc-per-node 4 --master-port $port bench.py --gpus 4 --config c9 $extra --steps 10 \
            --warmup 3 --no-e2e --no-cpu-baseline > "gpurun_out/table_c9_${tag}_n4.json" 2> /dev/null
        tail -c 300 "gpurun_out/table_c9_${tag}_n4.json" >> gpurun_out/final_table_n4.txt
    done
    bash "$0" scale 4
    echo "final4 done ($rev)" ;;
*)
    echo "unknown recipe $recipe"; exit 2 ;;
esac
