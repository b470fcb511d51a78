#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full captures.
# Usage (under gpurun): bash tools/gpu_round.sh <tag> [parts...]
# parts: tests smoke bench ncu  (default: all)
set -u
TAG=${1:-r01}; shift || true
PARTS=${*:-"tests smoke bench ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt
for p in $PARTS; do
  case $p in
    tests) timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/status.txt ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/status.txt ;;
    bench) timeout 900 python bench.py > $OUT/bench.txt 2>&1; echo "bench rc=$?" >> $OUT/status.txt ;;
    ab_lanes)
      for L in 1 2; do BODE_LANES=$L timeout 600 python bench.py --no-e2e --no-cpu --steps 5 > $OUT/bench_lanes$L.txt 2>&1; done
      echo "ab_lanes rc=$?" >> $OUT/status.txt ;;
    ncu_rkc)
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Heat \
        -s 1 -c 1 -o $OUT/prof_rkc python bench.py --steps 2 --warmup 1 --systems 4096 \
        --rkc-systems 131072 --no-e2e --no-cpu > $OUT/ncu_full_rkc.txt 2>&1
      echo "ncu_rkc rc=$?" >> $OUT/status.txt ;;
    ncu_exact)
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Pleiades \
        -s 1 -c 1 -o $OUT/prof_rkck_exact python bench.py --arith exact --steps 1 --warmup 1 --systems 262144 \
        --no-secondary --no-e2e --no-cpu > $OUT/ncu_full_rkck_exact.txt 2>&1
      echo "ncu_exact rc=$?" >> $OUT/status.txt ;;
    diverge)
      timeout 600 python tools/divergence.py --problem pleiades > $OUT/diverge_pleiades.txt 2>&1
      timeout 600 python tools/divergence.py --problem heat --num 262144 --arith exact > $OUT/diverge_heat.txt 2>&1
      timeout 600 python tools/divergence.py --problem expdecay --num 1048576 --arith exact > $OUT/diverge_expdecay.txt 2>&1
      timeout 600 python tools/divergence.py --problem expdecay_sorted --num 1048576 --arith exact > $OUT/diverge_expdecay_sorted.txt 2>&1
      echo "diverge rc=$?" >> $OUT/status.txt ;;
    ab_persist)
      timeout 600 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/bench_static.txt 2>&1
      for T in 4 8 16; do BODE_REFILL_MIN=$T timeout 600 python bench.py --persistent --no-e2e --no-cpu --no-secondary > $OUT/bench_persistent$T.txt 2>&1; done
      echo "ab_persist rc=$?" >> $OUT/status.txt ;;
    tfast) timeout 900 python -m pytest tests -x -q -m gpu -k "fast or persistent or block_size" > $OUT/pytest_fast.txt 2>&1; echo "tfast rc=$?" >> $OUT/status.txt ;;
    qfast) timeout 600 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/quick_fast.txt 2>&1; echo "qfast rc=$?" >> $OUT/status.txt ;;
    ab_block)
      for B in 32 64 128; do timeout 600 python bench.py --no-e2e --no-cpu --no-secondary --block $B > $OUT/bench_block$B.txt 2>&1; done
      for B in 32 64; do timeout 600 python bench.py --no-e2e --no-cpu --no-secondary --block $B --persistent > $OUT/bench_pblock$B.txt 2>&1; done
      echo "ab_block rc=$?" >> $OUT/status.txt ;;
    ab_rkc)
      IFS=';' read -ra VS <<< "${AB_RKC_VARIANTS:-8 128;8 96;16 96;16 128}"
      for V in "${VS[@]}"; do set -- $V
        BODE_LANES=$1 BODE_MAXREG=$2 timeout 600 python bench.py --no-e2e --no-cpu --steps 5 --systems 1048576 --rkc-systems 1048576 > $OUT/bench_rkc_L$1_R$2.txt 2>&1; done
      for R in 96 80; do BODE_LANES=1 BODE_MAXREG=$R timeout 600 python bench.py --no-e2e --no-cpu --steps 5 --systems 1048576 --rkc-systems 1048576 > $OUT/bench_rkc_exp$R.txt 2>&1; done
      echo "ab_rkc rc=$?" >> $OUT/status.txt ;;
    ab_lib)  # this build against paper_1611_02274_b200/lib/ab/libbode_base.so, alternating
      I=0; for L in base new base new; do I=$((I+1))
        if [ $L = base ]; then LP=$PWD/paper_1611_02274_b200/lib/ab/libbode_base.so; else LP=; fi
        BODE_LIB_PATH=$LP timeout 600 python bench.py --no-e2e --no-cpu --steps 5 > $OUT/bench_ab${I}_$L.txt 2>&1; done
      echo "ab_lib rc=$?" >> $OUT/status.txt ;;
    ncu_late)
      for W in 0 9; do
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:Pleiades, double" \
        -s $W -c 1 -o $OUT/prof_rkck_w$W python bench.py --steps 10 --warmup 0 --systems 262144 \
        --no-secondary --no-e2e --no-cpu > $OUT/ncu_rkck_w$W.txt 2>&1; done
      echo "ncu_late rc=$?" >> $OUT/status.txt ;;
    e2e)
      timeout 300 python tools/pcie.py > $OUT/pcie.txt 2>&1
      timeout 600 python bench.py --no-secondary --no-cpu > $OUT/bench_e2e.txt 2>&1
      echo "e2e rc=$?" >> $OUT/status.txt ;;
    ncu_persist)
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:persistent" \
        -s 1 -c 1 -o $OUT/prof_persist_w1 python bench.py --steps 10 --warmup 0 --systems 1048576 --persistent \
        --no-secondary --no-e2e --no-cpu > $OUT/ncu_persist.txt 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:Pleiades, double" \
        -s 1 -c 1 -o $OUT/prof_static_w1 python bench.py --steps 10 --warmup 0 --systems 1048576 \
        --no-secondary --no-e2e --no-cpu > $OUT/ncu_static.txt 2>&1
      echo "ncu_persist rc=$?" >> $OUT/status.txt ;;
    strag) timeout 600 python tools/straggler_sim.py > $OUT/straggler.txt 2>&1; echo "strag rc=$?" >> $OUT/status.txt ;;
    sweep) timeout 1500 python tools/sweep.py > $OUT/sweep.txt 2>&1; echo "sweep rc=$?" >> $OUT/status.txt ;;
    multirank)
      BODE_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
        --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 \
        --systems 262144 --rkc-systems 65536 --no-cpu > $OUT/bench_2rank.txt 2>&1
      echo "multirank bode rc=$?" >> $OUT/status.txt
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
        --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 3 \
        --warmup 3 --cpu-sample 4096 > $OUT/bench_2rank_ref.txt 2>&1
      echo "multirank ref rc=$?" >> $OUT/status.txt ;;
    texact) timeout 1500 python -m pytest tests -x -q -m gpu -k "exact or golden or kats or pleiades or stride or variant or cpp" > $OUT/pytest_exact.txt 2>&1; echo "texact rc=$?" >> $OUT/status.txt ;;
    qexact) timeout 600 python bench.py --arith exact --no-e2e --no-cpu --no-secondary > $OUT/quick_exact.txt 2>&1; echo "qexact rc=$?" >> $OUT/status.txt ;;
    ab_exact_lanes)
      for L in 1 2; do BODE_LANES=$L timeout 600 python bench.py --arith exact --no-e2e --no-cpu --no-secondary > $OUT/bench_exact_lanes$L.txt 2>&1; done
      echo "ab_exact_lanes rc=$?" >> $OUT/status.txt ;;
    qrkc) timeout 900 python bench.py --no-e2e --no-cpu --steps 10 --systems 65536 > $OUT/quick_rkc.txt 2>&1; echo "qrkc rc=$?" >> $OUT/status.txt ;;
    ab_heatblk)
      for V in "128 128" "112 64" "112 128" "128 64"; do set -- $V
        BODE_LANES=8 BODE_MAXREG=$1 timeout 600 python bench.py --no-e2e --no-cpu --steps 5 --systems 65536 --rkc-systems 1048576 --block $2 > $OUT/bench_heat_R$1_B$2.txt 2>&1; done
      echo "ab_heatblk rc=$?" >> $OUT/status.txt ;;
    phase)
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_1611_02274_b200/csrc \
        -DBODE_PHASE_TIMING tools/phase_probe.cu -o /tmp/phase_probe > $OUT/phase_build.txt 2>&1
      timeout 300 /tmp/phase_probe > $OUT/phase.txt 2>&1
      echo "phase rc=$?" >> $OUT/status.txt ;;
    quick)
      timeout 600 python bench.py --no-e2e --no-cpu --no-secondary > $OUT/quick_fast.txt 2>&1
      timeout 600 python bench.py --arith exact --no-e2e --no-cpu --no-secondary > $OUT/quick_exact.txt 2>&1
      echo "quick rc=$?" >> $OUT/status.txt ;;
    bench_exact) timeout 900 python bench.py --arith exact --no-cpu > $OUT/bench_exact.txt 2>&1; echo "bench_exact rc=$?" >> $OUT/status.txt ;;
    ncu)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --systems 1048576 \
        --rkc-systems 262144 --no-e2e --no-cpu > $OUT/ncu_launches_bench.txt 2>&1
      echo "ncu_launches rc=$?" >> $OUT/status.txt
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Pleiades \
        -s 1 -c 1 -o $OUT/prof_rkck python bench.py --steps 1 --warmup 1 --systems 262144 \
        --no-secondary --no-e2e --no-cpu > $OUT/ncu_full_rkck.txt 2>&1
      echo "ncu_full_rkck rc=$?" >> $OUT/status.txt
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Heat \
        -s 1 -c 1 -o $OUT/prof_rkc python bench.py --steps 2 --warmup 1 --systems 4096 \
        --rkc-systems 131072 --no-e2e --no-cpu > $OUT/ncu_full_rkc.txt 2>&1
      echo "ncu_full_rkc rc=$?" >> $OUT/status.txt ;;
  esac
done
