import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line)
print(round(d["value"]/1e9,3), round(d["ms_per_step"],3), round(d["roofline"]["frac"],3), d["roofline"]["classes_ms"], round(d["e2e"]["value"]/1e9,3))
