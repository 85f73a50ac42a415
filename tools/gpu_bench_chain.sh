cd $GRAFT_REPO_ROOT
for v in default gl8; do
  if [ $v = gl8 ]; then export WP_LIB=$GRAFT_REPO_ROOT/tools/variants/gl8/libwpb200.so; fi
  timeout 300 python bench.py --config bench_chain --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-strong-cfg5 --no-parity 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$v\", d[\"ms_per_step\"], d[\"config\"][\"passes\"][0][:90])"
done
unset WP_LIB
python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 600 -k "fuser or matrix or golden or catalog" 2>&1 | tail -1
