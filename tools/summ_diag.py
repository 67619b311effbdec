import sys,json
L=[l for l in sys.stdin]
R=[json.loads(l) for l in L if l.startswith("{")]
print(" its",[r["it"] for r in R],"kry",sum(r["kry"] for r in R),"ls",sum(r["ls"] for r in R),"conv",all(r["conv"] for r in R),L[-1].strip())
