#!/bin/bash
for cfg in "vgg16 32" "resnet50 256"; do
 for ms in "2 0 1" "2 2 0" "2 0 0"; do
  timeout 40 python tools/dbg_inc.py $cfg $ms > /tmp/o.txt 2>&1; rc=$?
  echo "cfg=$cfg ms=$ms rc=$rc $(tail -2 /tmp/o.txt | cut -c1-250)"
 done
done
