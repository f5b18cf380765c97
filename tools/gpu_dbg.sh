#!/bin/bash
timeout 60 python tools/dbg_inc2.py vgg16 64 0 2>&1 | tail -6 | head -3
FO_INC_SERIAL=1 timeout 60 python tools/dbg_inc2.py vgg16 64 0 2>&1 | tail -6 | head -3
FO_INC_SERIAL=1 timeout 60 python tools/dbg_inc2.py vgg16 64 1 2>&1 | tail -6 | head -3
