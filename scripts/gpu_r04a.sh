for c in c2 c5 c3; do
timeout 300 python scripts/e2e_breakdown.py $c 2>&1 | tail -1
MACH_NO_GRAPH=1 timeout 300 python scripts/e2e_breakdown.py $c 2>&1 | tail -1
done
