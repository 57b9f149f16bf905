# pass-2 side stream (row multiset + counts/histogram beside the key stream): CTAs per SM and priority
for prio in 1 0; do for ctas in 1 2 4 8; do
  echo "prio=$prio ctas=$ctas $(RK_SIDE_PRIO=$prio RK_ROWS_CTAS=$ctas python tools/memo_parts.py 2>&1 | head -1)"
done; done
echo "serial $(RK_OVERLAP=0 python tools/memo_parts.py 2>&1 | head -1)"
