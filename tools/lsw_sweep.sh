for mb in 4 5 6; do echo "MINB=$mb"; CDB_LSW_MINB=$mb python tools/probe_big.py 4 1000000 zt 1 2>&1 | tail -1 | grep -o "'ls_step[^)]*)\|'ls_resid[^)]*)\|'rescan[^)]*)"; done
