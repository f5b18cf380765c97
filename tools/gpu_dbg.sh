#!/bin/bash
for cfg in "vgg16 32" "vgg16 4096" "resnet50 4096"; do
 for ms in "0 0 1" "1 1 1" "1 2 1" "1 0 1" "1 0 0" "2 0 1"; do
  timeout 40 python tools/dbg_inc.py $cfg $ms > /tmp/o.txt 2>&1; rc=$?
  echo "cfg=$cfg ms=$ms rc=$rc $(tail -1 /tmp/o.txt | cut -c1-150)"
 done
done
