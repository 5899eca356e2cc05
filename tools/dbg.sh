#!/bin/bash
python tools/dbg_k2.py C3 gpus=8,n_f=100,n_i=30,n_u=10 2>&1 | head -12
