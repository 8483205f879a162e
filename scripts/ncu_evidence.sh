#!/bin/bash
# ncu --set full captures of the in-solve kernels (eager PCG solve, rdr_options.loop
# = RDR_LOOP_EAGER, scripts/prof_kernels.py --mode solve, selected by its NVTX range so
# that setup's autotuning launches of the same kernels are not picked) per config: the
# fused PCG-mode apply of iteration 1, the update + Jacobi, the patch kernel of iteration 1. Run under gpurun, one
# GPU. The reports are summarised on the box (gpurun_out/ must stay under 64 MiB):
#   gpurun_out/TAG_<cfg>_<kernel>.txt   metrics + warp-stall shares (scripts/ncu_summary.py full)
#   gpurun_out/TAG_<cfg>_<kernel>_src.txt  hottest SASS lines (scripts/ncu_summary.py source)
#   gpurun_out/TAG_traffic.json         dram bytes per launch (scripts/ncu_summary.py traffic)
#   bash scripts/ncu_evidence.sh TAG 3 4 5:12 2 6 7:10
#   KERNELS=patch bash scripts/ncu_evidence.sh TAG 3   (a subset of the kernels)
#   NCU_EXTRA='--cache-control none' ... (no L2 flush between replay passes: the in-solve state of
#   the L2-resident reference stack, which a flush turns into HBM reads)
TAG=$1; shift
mkdir -p gpurun_out
for spec in "$@"; do
  cfg=${spec%%:*}; p=${spec#*:}; [ "$p" = "$spec" ] && p=-
  name=cfg${cfg}; [ "$p" != "-" ] && name=${name}_p$p
  run="python scripts/prof_kernels.py $cfg $p 4 --mode solve"
  # APPLY_<name>=variant,slots,grid: profile the apply layout the bench ran (timing-based
  # autotuning under ncu's launch interception picks differently)
  ap=$(eval echo \${APPLY_${name}:-}); [ -n "$ap" ] && run="$run --apply $ap"
  $run > gpurun_out/${TAG}_${name}_plain.log 2>&1 || { echo "$name: plain run failed"; continue; }
  ncu_common="--set full --clock-control none --import-source on --kernel-name-base demangled --nvtx --nvtx-include solve/ ${NCU_EXTRA:-}"
  for k in ${KERNELS:-apply patch update}; do
    case $k in
      apply) sel='-k regex:apply_tc_kernel.*bool\)1 -s 1 -c 1' ;;
      patch) sel='-k regex:patch_(ldg|warp|warp_loop)_kernel -s 1 -c 1' ;;
      facta) sel='-k regex:fact_stage_a_kernel.*bool\)1 -s 1 -c 1' ;;
      factb) sel='-k regex:fact_stage_b_kernel.*bool\)1 -s 1 -c 1' ;;
      update) sel='-k regex:pcg_update_jacobi -s 1 -c 1' ;;
    esac
    rep=/tmp/${TAG}_${name}_${k}
    timeout 900 ncu $ncu_common $sel -o $rep -f $run > gpurun_out/${TAG}_${name}_${k}_ncu.log 2>&1
    if [ -f $rep.ncu-rep ]; then
      python scripts/ncu_summary.py full $rep.ncu-rep > gpurun_out/${TAG}_${name}_${k}.txt 2>&1
      python scripts/ncu_summary.py source $rep.ncu-rep > gpurun_out/${TAG}_${name}_${k}_src.txt 2>&1
      python scripts/ncu_summary.py traffic $rep.ncu-rep $name gpurun_out/${TAG}_traffic.json >> gpurun_out/${TAG}_traffic.log 2>&1
      rm -f $rep.ncu-rep
    fi
  done
  echo "$name done"
done
