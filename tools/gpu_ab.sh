python tools/kbench.py
FKD_REG_MAXK=16 python tools/kbench.py
