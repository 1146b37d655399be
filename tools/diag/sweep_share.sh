for cfg in "0 0" "2 2" "3 1" "2 1" "1 2" "3 2" "4 1"; do
  set -- $cfg
  echo "== chunk_share=$1 seg_share=$2"
  HDP_CHUNK_SHARE=$1 HDP_SEG_SHARE=$2 python tools/agg_ab.py 7 c5 2>&1 | tail -1
done
echo "== seg_prio=0"; HDP_SEG_PRIO=0 python tools/agg_ab.py 7 c5 2>&1 | tail -1
python tools/c4_reps.py c4_hdp 8
