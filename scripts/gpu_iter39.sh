cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 8 16 32; do echo "chunks=$k" >> gpurun_out/e2e.log; TOOM_HOST_CHUNKS=$k timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c4 | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(d['e2e'])" >> gpurun_out/e2e.log 2>&1; done
