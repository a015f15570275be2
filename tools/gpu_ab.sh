for cfg in "8 4" "8 6" "12 4" "12 6" "16 6" "16 8"; do set -- $cfg; echo "div $1 streams $2"; FKD_CHUNK_DIV=$1 FKD_STREAMS=$2 python tools/e2e_diag.py 2>&1 | sed -n 2p; done
