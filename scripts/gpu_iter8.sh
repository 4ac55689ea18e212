timeout 300 python scripts/diag_mha.py 4 2
timeout 300 python scripts/diag_mha.py 16 20
bash scripts/ab.sh ab/a .
