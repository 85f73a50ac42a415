# chain_lb A/B: default build vs every variant in tools/variants, on cfg3 and a cfg5 slice, REPS times
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
o=gpurun_out/lb_ab.txt
: > $o
for rep in $(seq ${REPS:-2}); do
  for cfg in ${CFGS:-cfg3 cfg5}; do
    for v in default $(ls tools/variants 2>/dev/null); do
      if [ $v = default ]; then L=""; else L=tools/variants/$v/libwpb200.so; fi
      t=$(WP_LIB=$L timeout 300 python tools/trace_lb.py $cfg 2>&1 | grep "ms per pass" | awk '{print $NF}')
      echo "$cfg $v $t" >> $o
    done
  done
done
cat $o
