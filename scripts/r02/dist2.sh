set -u
for rs in 16 32; do TM_LOOPBACK_RESERVE=$rs timeout 900 python scripts/scaling_projection.py 2>&1 | grep -v "^{" ; done
