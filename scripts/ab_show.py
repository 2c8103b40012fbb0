import json, sys
lab = "(run)"
for l in open(sys.argv[1]):
    if l.startswith('=='):
        lab = l.strip()
    elif l.startswith('{'):
        d = json.loads(l)
        k = d['kernels']
        print(f"{lab:40s} fps {d['value']:7.1f}  march {k['march_ms']:.3f} ms  build {k['build_ms']:.3f} ms  Gs/s {d['gsamples_per_s']:.1f}")
    elif l.strip():
        print("   ", l.strip()[:240])
