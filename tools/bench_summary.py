import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["ms_per_step"],4), {k:v["ms_per_launch"] for k,v in d["breakdown"].items()}, d.get("fp64_fallback_entries"))
    except Exception as e: print(f, "ERR", e)
