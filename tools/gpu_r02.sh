#!/bin/bash
# Round-2 GPU session helper. Usage (under gpurun): bash tools/gpu_r02.sh <tag> [parts...]
set -u
TAG=${1:-r02}; shift || true
PARTS=${*:-"tests bench"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt
for p in $PARTS; do
  case $p in
    tests) timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/status.txt ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/status.txt ;;
    bench) S=$(date +%s); timeout 1700 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench.txt 2> $OUT/bench.err; echo "bench rc=$? wall=$(( $(date +%s) - S ))s" >> $OUT/status.txt ;;
    ref) timeout 600 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref.txt 2>&1; echo "ref rc=$?" >> $OUT/status.txt ;;
    multirank)
      BODE_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
        --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 12 --warmup 3 \
        --systems 1048576 --rkc-systems 65536 --aux-systems 65536 --no-cpu > $OUT/bench_2rank.txt 2>&1
      echo "multirank rc=$?" >> $OUT/status.txt ;;
  esac
done
# (appended parts; run with: bash tools/gpu_r02.sh <tag> ncu sanitize ...)
for p in $PARTS; do
  case $p in
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $OUT/launches.csv python bench.py --steps 20 --warmup 5 > $OUT/ncu_launches_bench.txt 2>&1
      echo "ncu_launches rc=$?" >> $OUT/status.txt
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Pleiades \
        -s 1 -c 1 -o $OUT/prof_rkck_fast python bench.py --steps 2 --warmup 1 --systems 16777216 \
        --no-secondary --no-e2e --no-cpu > $OUT/ncu_full_rkck_fast.txt 2>&1
      echo "ncu_rkck_fast rc=$?" >> $OUT/status.txt
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Pleiades \
        -s 1 -c 1 -o $OUT/prof_rkck_exact python bench.py --arith exact --steps 2 --warmup 1 --systems 4194304 \
        --no-secondary --no-e2e --no-cpu > $OUT/ncu_full_rkck_exact.txt 2>&1
      echo "ncu_rkck_exact rc=$?" >> $OUT/status.txt
      timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Heat \
        -s 1 -c 1 -o $OUT/prof_heat_exact python bench.py --steps 2 --warmup 1 --systems 4096 \
        --rkc-systems 4194304 --aux-systems 0 --no-e2e --no-cpu > $OUT/ncu_full_heat_exact.txt 2>&1
      echo "ncu_heat_exact rc=$?" >> $OUT/status.txt
      timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:Heat \
        -s 4 -c 1 -o $OUT/prof_heat_fast python bench.py --steps 2 --warmup 1 --systems 4096 \
        --rkc-systems 4194304 --aux-systems 0 --no-e2e --no-cpu > $OUT/ncu_full_heat_fast.txt 2>&1
      echo "ncu_heat_fast rc=$?" >> $OUT/status.txt ;;
    sanitize)
      for T in memcheck racecheck synccheck initcheck; do
        timeout 900 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_probe.py > $OUT/sanitize_$T.txt 2>&1
        echo "sanitize $T rc=$?" >> $OUT/status.txt
      done ;;
  esac
done
for p in $PARTS; do
  case $p in
    ab_sum)  # heat64 RKC with the new sums vs lib/ab/sum0 (BODE_RKC_SUM=0), alternating
      I=0; for V in sum0 new sum0 new; do I=$((I+1))
        if [ $V = new ]; then LP=; else LP=$PWD/paper_1611_02274_b200/lib/ab/$V/libbode.so; fi
        BODE_LIB_PATH=$LP timeout 600 python bench.py --steps 5 --warmup 1 --systems 4096 --rkc-systems 4194304 \
          --aux-systems 0 --no-e2e --no-cpu > $OUT/ab_sum_${I}_$V.txt 2>&1; done
      echo "ab_sum rc=$?" >> $OUT/status.txt ;;
    trkc) timeout 900 python -m pytest tests -x -q -m gpu -k "heat or rkc or stiff or expdecay or brusselator or user" -s > $OUT/pytest_rkc.txt 2>&1; echo "trkc rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    lat) [ -x tools/fp64_latency ] && timeout 120 tools/fp64_latency > $OUT/fp64_latency.json 2>&1; echo "lat rc=$?" >> $OUT/status.txt ;;
  esac
done
# ncu with on-box post-processing: only summaries come back (gpurun_out <= 64 MiB)
for p in $PARTS; do
  case $p in
    ncu2)
      NCUP=/tmp/ncu_$TAG; mkdir -p $NCUP
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $NCUP/launches.csv python bench.py --steps 20 --warmup 5 > $OUT/ncu_launches_bench.txt 2>&1
      echo "ncu_launches rc=$?" >> $OUT/status.txt
      python tools/ncu_summary.py --launches $NCUP/launches.csv $OUT/launches > /dev/null 2>&1
      gzip -c $NCUP/launches.csv > $OUT/launches.csv.gz
      cap() {  # name regex skip systems args...
        local n=$1 k=$2 s=$3 sys=$4; shift 4
        timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
          -k regex:$k -s $s -c 1 -o $NCUP/$n python bench.py "$@" > $OUT/ncu_full_$n.txt 2>&1
        echo "ncu_$n rc=$?" >> $OUT/status.txt
        python tools/ncu_lines.py $NCUP/$n.ncu-rep 60 > $OUT/lines_$n.txt 2>&1
        SPECS="$SPECS $n=$NCUP/$n.ncu-rep:$sys"
      }
      SPECS=""
      cap rkck_fast Pleiades 1 16777216 --steps 2 --warmup 1 --systems 16777216 --no-secondary --no-e2e --no-cpu
      cap rkck_exact Pleiades 1 4194304 --arith exact --steps 2 --warmup 1 --systems 4194304 --no-secondary --no-e2e --no-cpu
      cap heat_exact Heat 1 4194304 --steps 2 --warmup 1 --systems 4096 --rkc-systems 4194304 --aux-systems 0 --no-e2e --no-cpu
      cap heat_fast Heat 4 4194304 --steps 2 --warmup 1 --systems 4096 --rkc-systems 4194304 --aux-systems 0 --no-e2e --no-cpu
      python tools/ncu_summary.py $OUT/ncu $SPECS > $OUT/ncu_summary.txt 2>&1
      echo "ncu_summary rc=$?" >> $OUT/status.txt
      ls -la $NCUP > $OUT/ncu_reports_ls.txt ;;
    newtests) timeout 1200 python -m pytest tests -x -q -m gpu -k "wide or budget or fixed" > $OUT/pytest_new.txt 2>&1; echo "newtests rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    ab_ctrl)  # RKC controller scalars in shared memory (new) vs registers (lib/ab/ctrl0), alternating
      I=0; for V in ctrl0 nobudget new ctrl0 nobudget new; do I=$((I+1))
        if [ $V = new ]; then LP=; else LP=$PWD/paper_1611_02274_b200/lib/ab/$V/libbode.so; fi
        BODE_LIB_PATH=$LP timeout 600 python bench.py --steps 5 --warmup 1 --systems 4096 --rkc-systems 4194304 \
          --aux-systems 4194304 --no-e2e --no-cpu > $OUT/ab_ctrl_${I}_$V.txt 2>&1; done
      echo "ab_ctrl rc=$?" >> $OUT/status.txt ;;
    ncuheat)
      NCUP=/tmp/ncu_$TAG; mkdir -p $NCUP
      timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k regex:Heat -s 1 -c 1 -o $NCUP/heat_exact python bench.py --steps 2 --warmup 1 --systems 4096 \
        --rkc-systems 4194304 --aux-systems 0 --no-e2e --no-cpu > $OUT/ncu_full_heat_exact.txt 2>&1
      echo "ncuheat rc=$?" >> $OUT/status.txt
      python tools/ncu_lines.py $NCUP/heat_exact.ncu-rep 60 > $OUT/lines_heat_exact.txt 2>&1
      python tools/ncu_summary.py $OUT/ncu_heat heat_exact=$NCUP/heat_exact.ncu-rep:4194304 > /dev/null 2>&1 ;;
  esac
done
for p in $PARTS; do
  case $p in
    ab_budget)  # attempt-budget countdown (new) vs compiled out (lib/ab/nobudget), full default sizes
      I=0; for V in nobudget new nobudget new; do I=$((I+1))
        if [ $V = new ]; then LP=; else LP=$PWD/paper_1611_02274_b200/lib/ab/$V/libbode.so; fi
        BODE_LIB_PATH=$LP timeout 900 python bench.py --steps 5 --warmup 1 --no-e2e --no-cpu > $OUT/ab_budget_${I}_$V.txt 2>&1; done
      echo "ab_budget rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    ab_chunks)  # host-pointer pipeline depth: 32 (default) vs 64 / 128 chunks, e2e only matters
      I=0; for V in new chunks64 chunks128 new chunks64 chunks128; do I=$((I+1))
        if [ $V = new ]; then LP=; else LP=$PWD/paper_1611_02274_b200/lib/ab/$V/libbode.so; fi
        BODE_LIB_PATH=$LP timeout 900 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu > $OUT/ab_chunks_${I}_$V.txt 2>&1; done
      echo "ab_chunks rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    ab_stats)  # 40-byte stats over PCIe (new) vs 64-byte records (lib/ab/fullstats): e2e
      I=0; for V in fullstats new fullstats new fullstats new; do I=$((I+1))
        if [ $V = new ]; then LP=; else LP=$PWD/paper_1611_02274_b200/lib/ab/$V/libbode.so; fi
        BODE_LIB_PATH=$LP timeout 900 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu > $OUT/ab_stats_${I}_$V.txt 2>&1; done
      echo "ab_stats rc=$?" >> $OUT/status.txt ;;
    tcompact) timeout 1200 python -m pytest tests -x -q -m gpu -k "compact or shards or budget" > $OUT/pytest_compact.txt 2>&1; echo "tcompact rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    pcie) timeout 600 python tools/pcie.py --num 16777216 --stats-sweep > $OUT/pcie_sweep.json 2>&1; echo "pcie rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    widebench) timeout 900 python tests/experiments/wide_bench.py > $OUT/wide_bench.jsonl 2> $OUT/wide_bench.err; echo "widebench rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    variants)  # compiled lane/register variants of the RKC kernels, current code (BODE_LANES / BODE_MAXREG)
      for V in "0 -1" "8 112" "8 168" "4 168" "4 255" "8 128" "0 -1"; do set -- $V
        BODE_LANES=$1 BODE_MAXREG=$2 timeout 600 python bench.py --steps 5 --warmup 1 --systems 4096 \
          --rkc-systems 4194304 --aux-systems 4194304 --no-e2e --no-cpu > $OUT/variant_L$1_R$2_$RANDOM.txt 2>&1
      done
      echo "variants rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    ab_skew)  # EXACT sum-chain scratch skewed per half-warp (new) vs not (lib/ab/noskew)
      I=0; for V in noskew new noskew new; do I=$((I+1))
        if [ $V = new ]; then LP=; else LP=$PWD/paper_1611_02274_b200/lib/ab/$V/libbode.so; fi
        BODE_LIB_PATH=$LP timeout 600 python bench.py --steps 5 --warmup 1 --systems 4096 --rkc-systems 4194304 \
          --aux-systems 4194304 --no-e2e --no-cpu > $OUT/ab_skew_${I}_$V.txt 2>&1; done
      echo "ab_skew rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    pvariants)  # Pleiades FAST: one lane (RKN) vs the axis-split lane pair
      for V in 0 2 0 2; do
        BODE_LANES=$V timeout 600 python bench.py --steps 10 --warmup 3 --no-secondary --no-e2e --no-cpu > $OUT/pvariant_L${V}_$RANDOM.txt 2>&1
      done
      echo "pvariants rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    ab_cbrt)  # FAST cube root: MUFU seed + Newton (new) vs libdevice cbrt (lib/ab/libcbrt)
      I=0; for V in libcbrt new libcbrt new; do I=$((I+1))
        if [ $V = new ]; then LP=; else LP=$PWD/paper_1611_02274_b200/lib/ab/$V/libbode.so; fi
        BODE_LIB_PATH=$LP timeout 600 python bench.py --steps 5 --warmup 1 --systems 4096 --rkc-systems 4194304 \
          --aux-systems 4194304 --no-e2e --no-cpu > $OUT/ab_cbrt_${I}_$V.txt 2>&1; done
      echo "ab_cbrt rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    ab_sqrt)  # FAST sqrt: rsqrt seed + correction (new) vs libdevice sqrt (lib/ab/libsqrt)
      I=0; for V in libsqrt new libsqrt new; do I=$((I+1))
        if [ $V = new ]; then LP=; else LP=$PWD/paper_1611_02274_b200/lib/ab/$V/libbode.so; fi
        BODE_LIB_PATH=$LP timeout 600 python bench.py --steps 5 --warmup 1 --systems 4096 --rkc-systems 4194304 \
          --aux-systems 4194304 --no-e2e --no-cpu > $OUT/ab_sqrt_${I}_$V.txt 2>&1; done
      echo "ab_sqrt rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    ab_rkn)  # FAST Pleiades on the spill-free budget instance (new) vs the plain instance (lib/ab/rknplain)
      I=0; for V in rknplain new rknplain new rknplain new; do I=$((I+1))
        if [ $V = new ]; then LP=; else LP=$PWD/paper_1611_02274_b200/lib/ab/$V/libbode.so; fi
        BODE_LIB_PATH=$LP timeout 600 python bench.py --steps 20 --warmup 5 --no-secondary --no-e2e --no-cpu > $OUT/ab_rkn_${I}_$V.txt 2>&1; done
      echo "ab_rkn rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    ncufast)  # the headline kernel only: full capture at 2^24 + launch list, summarised on the box
      NCUP=/tmp/ncu_$TAG; mkdir -p $NCUP
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $NCUP/launches.csv python bench.py --steps 20 --warmup 5 > $OUT/ncu_launches_bench.txt 2>&1
      echo "ncu_launches rc=$?" >> $OUT/status.txt
      python tools/ncu_summary.py --launches $NCUP/launches.csv $OUT/launches > /dev/null 2>&1
      gzip -c $NCUP/launches.csv > $OUT/launches.csv.gz
      timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k regex:Pleiades -s 1 -c 1 -o $NCUP/rkck_fast python bench.py --steps 2 --warmup 1 --systems 16777216 \
        --no-secondary --no-e2e --no-cpu > $OUT/ncu_full_rkck_fast.txt 2>&1
      echo "ncu_rkck_fast rc=$?" >> $OUT/status.txt
      python tools/ncu_lines.py $NCUP/rkck_fast.ncu-rep 60 > $OUT/lines_rkck_fast.txt 2>&1
      python tools/ncu_summary.py $OUT/ncu rkck_fast=$NCUP/rkck_fast.ncu-rep:16777216 > $OUT/ncu_summary.txt 2>&1 ;;
  esac
done
for p in $PARTS; do
  case $p in
    ab_div)  # FAST controller/power-method division via rcp_fast (new) vs IEEE division (lib/ab/ieeediv)
      I=0; for V in ieeediv new ieeediv new; do I=$((I+1))
        if [ $V = new ]; then LP=; else LP=$PWD/paper_1611_02274_b200/lib/ab/$V/libbode.so; fi
        BODE_LIB_PATH=$LP timeout 600 python bench.py --steps 5 --warmup 1 --systems 4096 --rkc-systems 4194304 \
          --aux-systems 4194304 --no-e2e --no-cpu > $OUT/ab_div_${I}_$V.txt 2>&1; done
      echo "ab_div rc=$?" >> $OUT/status.txt ;;
  esac
done
for p in $PARTS; do
  case $p in
    exp_treesum)  # experiment: EXACT heat64 with tree sums (not bitwise) -- how much the sequential chain costs
      I=0; for V in treesum new treesum new; do I=$((I+1))
        if [ $V = new ]; then LP=; else LP=$PWD/paper_1611_02274_b200/lib/ab/$V/libbode.so; fi
        BODE_LIB_PATH=$LP timeout 600 python bench.py --steps 5 --warmup 1 --systems 4096 --rkc-systems 4194304 \
          --aux-systems 0 --no-e2e --no-cpu > $OUT/exp_treesum_${I}_$V.txt 2>&1; done
      echo "exp_treesum rc=$?" >> $OUT/status.txt ;;
  esac
done
