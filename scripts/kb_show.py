import json
import sys
name = "-"
for line in open(sys.argv[1]):
    line = line.strip()
    if line.startswith('{'):
        d = json.loads(line)
        print(f"{name:10s}", ' '.join(f"s{k}: f{v['fwd_ms']:.3f} b{v['bwd_ms']:.3f}" for k, v in d.items()))
    elif line:
        name = line
