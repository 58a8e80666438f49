"""Print the headline numbers of a gpurun_out bench log and the full-search JSONs (usage: show.py TAG)."""
import json
import sys

tag = sys.argv[1]
for line in open(f"gpurun_out/bench_{tag}.log"):
    if line.startswith("{"):
        d = json.loads(line)
        print("sweep ms", round(d["ms_per_step"], 3), "phases", {k: round(v, 3) for k, v in d["phase_ms"].items()},
              "e2e ms", round(d["e2e"]["ms_per_step"], 3), "clocks", d["clocks"]["sm_mhz"])
for w in ["gpt96", "gpt96-bmw", "swin-bmw", "vit-bmw", "bert", "t5-16"]:
    try:
        d = json.load(open(f"gpurun_out/fs_{w}{sys.argv[2] if len(sys.argv) > 2 else ''}.json"))
        print(w, round(d["ms_per_step"], 2), "device", round(d.get("device_ms", 0), 2))
    except Exception as ex:  # noqa: BLE001
        print(w, "?", ex)
