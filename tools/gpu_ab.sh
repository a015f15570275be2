for s in 3 4; do for d in 4 6 8; do echo "streams $s div $d $(FKD_STREAMS=$s FKD_CHUNK_DIV=$d python tools/e2e_diag.py 2>&1 | grep -E 'auto')"; done; done
