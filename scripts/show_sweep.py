"""Print harness sweep JSON files as one row per (flavor, size)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    print("==", f)
    for k, v in d.items():
        if not isinstance(v, list):
            continue
        for x in v:
            print(f"{k[:8]:8s} {x.get('bytes'):>11} rt {x['us_per_round']:8.1f} "
                  f"b2b {x.get('us_per_round_b2b', 0):8.1f} pipe {x.get('us_per_round_pipelined', 0):8.1f} "
                  f"bw {x['busbw_gbs']:5.0f}/{x.get('busbw_b2b_gbs', 0):5.0f}/"
                  f"{x.get('busbw_pipelined_gbs', 0):5.0f} dev {x.get('busbw_device_gbs') or 0:5.0f}")
