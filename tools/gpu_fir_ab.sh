# fir_tc A/B on a config (default cfg2): every built variant's time per pass + output check;
# variants named *tr* (built with -DFT_TRACE) also print the stage timeline
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
o=gpurun_out/fir_ab.txt
: > $o
for rep in $(seq ${REPS:-1}); do for v in default $(ls tools/variants); do
  for nin in ${NINS:-3}; do
    echo "== $v $(cat tools/variants/$v/flags.txt 2>/dev/null) WP_FIR_NIN=$nin" >> $o
    if [ $v = default ]; then L=""; else L=tools/variants/$v/libwpb200.so; fi
    case $v in
      *tr*) WP_FIR_NIN=$nin WP_LIB=$L timeout 300 python tools/trace_fir.py ${1:-cfg2} >> $o 2>&1 ;;
      *) WP_FIR_NIN=$nin WP_LIB=$L timeout 300 python tools/trace_fir.py ${1:-cfg2} 2>&1 | grep "ms per pass\|err\|fir_tc\[" >> $o ;;
    esac
  done
done; done
cat $o
