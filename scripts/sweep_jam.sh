for j in 0 2 4 8 16; do MAPC_JAM=$j timeout 300 python scripts/probe_direct5a.py 2>&1 | grep '^{' ; done
