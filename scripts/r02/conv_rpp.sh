# Direct conv: filter rows per pass (TM_CONV_RPP caps it; smaller passes = more, smaller TMEM
# A slots, so the split can run further ahead of the MMAs) -- parity and time per setting.
for r in 0 2 1; do
  TM_CONV_RPP=$r timeout 300 python -m pytest tests/test_conv.py -q -x -p no:cacheprovider -k "direct or paper_shape" 2>&1 | tail -1
done
for i in 1 2; do
  for r in 0 2 1; do
    TM_CONV_RPP=$r bash scripts/ms.sh "conv3 rpp<=$r" --config CONV --steps 20 --warmup 5 --no-cpu
    TM_CONV_RPP=$r bash scripts/ms.sh "conv5 rpp<=$r" --config CONV --conv-r 5 --steps 20 --warmup 5 --no-cpu
  done
done
