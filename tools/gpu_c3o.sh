cd "$(dirname "$0")/.."
timeout 120 python tools/c3_prof.py cfg3 2 > /dev/null || { echo hung; exit 1; }
for d in 0; do
  echo "== dbg $d"
  WP_CT_DBG=$d timeout 100 python tools/trace_c3.py cfg3 | grep -E "span|opfull -> mma0|mma0 -> mma1|epi0 -> epi1|conv0 -> opfull|period of  conv0"
done
