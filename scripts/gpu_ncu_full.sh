# full ncu capture of one kernel (regex $1) of one C2 step
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/prof_c2.py 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -c 1 -o gpurun_out/prof_$2 python scripts/prof_c2.py 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log
