python tools/repro_proj.py 2>&1 | tail -12
python tools/repro_c6.py 2>&1 | tail -5
PCY_K3PAR=0 python tools/repro_c6.py 2>&1 | tail -5
