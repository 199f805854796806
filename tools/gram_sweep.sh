for w in 2 3 4 6 8; do echo "WPB=$w"; CDB_GRAM_WPB=$w python tools/probe_big.py 4 1000000 zt 1 2>&1 | tail -1 | grep -o "gram_step2[^)]*)"; done
