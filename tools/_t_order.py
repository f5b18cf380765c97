import sys, os
sys.argv = ["x", "resnet50", "4096"]
exec(open("tools/time_inc.py").read().split("out = {")[0])
print("m1s0", timed(1, 0))
print("m1s0", timed(1, 0))
print("m1s1", timed(1, 1))
print("m1s0", timed(1, 0))
print("m1s2", timed(1, 2))
print("m1s0", timed(1, 0))
print("m0s0", timed(0, 0))
print("m1s0", timed(1, 0))
