# One GPU session of measurements, each leg under its own timeout, logs into
# gpurun_out/<tag>_*.  Usage (from the repo root, on the GPU box):
#   bash tools/gpu_session.sh <tag> <leg> [<leg> ...]
# legs: probe (DSMEM dQ reduce probe), bench (C2 N=1), c3, c4, c5 (Lkv sweeps /
#       layer stack at N=1), bench_n / c3_n / c4_n / c5_n / c5small_n (all
#       visible GPUs, torchrun), launches / launches_c4 (ncu launch lists),
#       ncu_full / ncu_fwd_dq (ncu --set full of the hot kernels), kernels /
#       hbm / gemm / recompute (kernel-level rates), p2p / ce (transport
#       probes), fullscale_n (n-way vs 1-way at full C2 size), guards,
#       sanitize, pytest / pytest_multi / pytest_gemm (pytest -m gpu subsets)
set -u
tag=$1; shift
out=gpurun_out
mkdir -p $out
python -m paper_2502_02406_b200.build > $out/${tag}_build.log 2>&1 || { echo "build failed"; exit 1; }
nvidia-smi -q -d CLOCK,PERFORMANCE > $out/${tag}_clocks_before.txt 2>&1
for leg in "$@"; do
  t0=$(date +%s)
  case $leg in
    probe)
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/dqprobe \
        tools/dq_cluster_reduce_probe.cu > $out/${tag}_probe_build.log 2>&1 &&
      timeout 120 /tmp/dqprobe > $out/${tag}_probe.jsonl 2>&1 ;;
    bench)
      timeout 600 python bench.py --steps 10 --warmup 3 > $out/${tag}_bench_c2.json 2> $out/${tag}_bench_c2.err ;;
    c3)
      timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-e2e \
        > $out/${tag}_bench_c3.json 2> $out/${tag}_bench_c3.err ;;
    c4)
      timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu \
        > $out/${tag}_bench_c4.json 2> $out/${tag}_bench_c4.err ;;
    c5)
      timeout 1200 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu --no-e2e \
        > $out/${tag}_bench_c5.json 2> $out/${tag}_bench_c5.err ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file $out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu \
        > $out/${tag}_launches.log 2>&1 ;;
    bench_n)   # all visible GPUs, torchrun, C2 (BENCH_SKV overrides Lkv)
      n=$(nvidia-smi -L | wc -l)
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 29517 bench.py --gpus $n --steps 10 --warmup 3 ${BENCH_SKV:+--skv $BENCH_SKV} \
        > $out/${tag}_bench_n${n}${BENCH_SKV:+_skv$BENCH_SKV}.json 2> $out/${tag}_bench_n${n}.err ;;
    c3_n)
      n=$(nvidia-smi -L | wc -l)
      timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 29521 bench.py --gpus $n --workload c3 --steps 3 --warmup 3 --no-e2e \
        > $out/${tag}_bench_c3_n${n}.json 2> $out/${tag}_bench_c3_n${n}.err ;;
    c4_n)
      n=$(nvidia-smi -L | wc -l)
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 29522 bench.py --gpus $n --workload c4 --steps 10 --warmup 3 --no-e2e \
        > $out/${tag}_bench_c4_n${n}.json 2> $out/${tag}_bench_c4_n${n}.err ;;
    c5small_n)
      n=$(nvidia-smi -L | wc -l)
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 29523 bench.py --gpus $n --workload c5 --sweep 65536,262144 --steps 5 --warmup 3 --no-e2e \
        > $out/${tag}_bench_c5small_n${n}.json 2> $out/${tag}_bench_c5small_n${n}.err ;;
    c5_n)
      n=$(nvidia-smi -L | wc -l)
      timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 29518 bench.py --gpus $n --workload c5 --steps 3 --warmup 3 --no-e2e \
        > $out/${tag}_bench_c5_n${n}.json 2> $out/${tag}_bench_c5_n${n}.err ;;
    sanitize)
      for tool in memcheck racecheck synccheck; do
        timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py \
          > $out/${tag}_sanitize_$tool.log 2>&1
        echo "sanitize $tool exit=$?" >> $out/${tag}_legs.txt
      done ;;
    launches_c4)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
        --log-file $out/${tag}_launches_c4.csv python bench.py --workload c4 --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph \
        > $out/${tag}_launches_c4.log 2>&1 ;;
    ncu_fwd_dq)   # --set full of the forward and dQ launches of the C2 bench
      for kn in fwd_kernel bwd_dq_kernel; do
        timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kn -c 1 \
          -o $out/${tag}_ncu_$kn python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu \
          > $out/${tag}_ncu_$kn.log 2>&1
      done ;;
    ncu_full)   # one --set full capture per hot kernel
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_dkv_kernel -c 1 \
        -o $out/${tag}_ncu_dkv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu \
        > $out/${tag}_ncu_dkv.log 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16_kernel -c 2 \
        -o $out/${tag}_ncu_gemm python tools/gemm_probe.py --preset llama \
        > $out/${tag}_ncu_gemm.log 2>&1 ;;
    guards)
      timeout 600 python -m pytest tests/test_gpu_guards.py -q -s --timeout 300 -p no:cacheprovider \
        > $out/${tag}_guards.log 2>&1 ;;
    recompute)
      timeout 600 python tools/bench_recompute.py --preset flamingo > $out/${tag}_recompute_flamingo.json 2>&1
      timeout 600 python tools/bench_recompute.py --preset llama > $out/${tag}_recompute_llama.json 2>&1 ;;
    p2p)
      n=$(nvidia-smi -L | wc -l)
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 29519 tools/p2p_bw.py > $out/${tag}_p2p_n${n}.json 2> $out/${tag}_p2p.err ;;
    ce)
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29520 tools/ce_probe.py > $out/${tag}_ce_probe.json 2> $out/${tag}_ce_probe.err ;;
    kernels)   # kernel-level rates at round shapes
      for sh in c2round c4round c4gath c3round c2gath; do
        timeout 300 python tools/bench_kernels.py --shape $sh --bwd --bf16-grads >> $out/${tag}_kernels.jsonl 2>&1
      done ;;
    fullscale_n)
      n=$(nvidia-smi -L | wc -l)
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 29524 tools/fullscale_multi_check.py > $out/${tag}_fullscale_n${n}.json 2> $out/${tag}_fullscale.err
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port 29525 tools/nvlink_counters.py > $out/${tag}_nvlink_n${n}.json 2> $out/${tag}_nvlink.err ;;
    hbm)
      timeout 300 python tools/bench_hbm_kernels.py > $out/${tag}_hbm.json 2>&1 ;;
    gemm)
      timeout 300 python tools/gemm_probe.py --preset llama > $out/${tag}_gemm_llama.jsonl 2>&1
      timeout 300 python tools/gemm_probe.py --preset flamingo > $out/${tag}_gemm_flamingo.jsonl 2>&1 ;;
    pytest_gemm)
      timeout 900 python -m pytest tests/test_gpu_project.py tests/test_gpu_recompute.py tests/test_gpu_mllm.py -q -s --timeout 600 -p no:cacheprovider \
        > $out/${tag}_pytest_gemm.log 2>&1 ;;
    pytest)
      timeout 1800 python -m pytest tests -m gpu -q -s --timeout 600 -p no:cacheprovider \
        > $out/${tag}_pytest.log 2>&1 ;;
    pytest_multi)
      timeout 900 python -m pytest tests/test_gpu_multi.py -q -s --timeout 600 -p no:cacheprovider \
        > $out/${tag}_pytest_multi.log 2>&1 ;;
    *) echo "unknown leg $leg" ;;
  esac
  echo "$leg exit=$? secs=$(( $(date +%s) - t0 ))" | tee -a $out/${tag}_legs.txt
done
