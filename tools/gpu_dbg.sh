#!/bin/bash
timeout 60 python tools/dbg_inc2.py vgg16 64 0 2>&1 | tail -6 | head -2
timeout 60 python tools/dbg_inc2.py resnet50 1024 1 2>&1 | tail -6 | head -2
