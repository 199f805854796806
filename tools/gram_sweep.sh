# step-2 Gram kernel variants on cfg 4 (1M signals), 2 runs each
for v in ${VARIANTS:-"CDB_GRAM_CPS=2" "CDB_GRAM_CPS=3" "CDB_GRAM_CTA=0"}; do echo "$v"; env $v python tools/probe_big.py 4 1000000 zt 2 2>&1 | tail -2 | grep -o "gram_step2[^)]*)"; done
