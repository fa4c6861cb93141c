# Two output rows per tile at 5x5 (TM_CONV_RO=2 now allowed for 5-tap filters): parity
# (direct-kernel tests incl. the paper's shape, forced) and time vs the one-row default.
TM_CONV_RO=2 timeout 400 python -m pytest tests/test_conv.py -q -x -p no:cacheprovider 2>&1 | tail -1
python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import paper_1804_10694_b200 as tm
for ro in ("0", "2"):
    print(ro, tm.conv2d_plan_name(32, 512, 512, 16, 16, 5, 5, 2))
PY
for i in 1 2; do
  for ro in 0 2; do TM_CONV_RO=$ro bash scripts/ms.sh "conv5 ro=$ro" --config CONV --conv-r 5 --steps 20 --warmup 5 --no-cpu; done
done
