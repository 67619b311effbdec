"""Line-search statistics of the C5 bench rollout (DP_DEBUG=2 log on stderr):
accepted step lengths, trials per Newton iteration, pre-check rejections."""
import collections
import re
import sys

acc = collections.Counter()
trials = []
cur = 0
pen = 0
for line in open(sys.argv[1]):
    m = re.search(r"ls=(\d+) t=([0-9.e+-]+) pen=(\d) st=(\d+) rmax_try=([0-9.e+-]+|nan|inf) \(rmax=([0-9.e+-]+)\)", line)
    if m:
        cur += 1
        pen += int(m.group(3))
        if float(m.group(5)) < float(m.group(6)):
            acc[m.group(2)] += 1
            trials.append(cur)
            cur = 0
        continue
    if "[dp] it=" in line and cur:
        trials.append(-cur)   # previous line search ended without acceptance
        cur = 0
print("accepted t:", sorted(acc.items(), key=lambda x: -float(x[0])))
print("line searches:", len(trials), "trials:", sum(abs(t) for t in trials), "penetrating:", pen)
print("trials per line search:", collections.Counter(trials))
