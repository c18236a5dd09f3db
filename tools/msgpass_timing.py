"""The message pass alone at 10M agents (roofline.message_pass_roofline):
ms per launch and the fraction of measured HBM."""
import json
import sys
from pathlib import Path

sys.path.insert(0, ".")
from paper_2110_04421_b200.roofline import message_pass_roofline  # noqa: E402

peaks = json.loads(Path("MEASURED_PEAKS.json").read_text()) if Path("MEASURED_PEAKS.json").exists() else {}
r = message_pass_roofline(10_000_000, peak_gbps=float(peaks.get("hbm_gbs", 6531.9)))
print(f"ms {r['ms_median']:.4f} (min {r['ms_min']:.4f})  {r['achieved']:.0f} GB/s  frac {r['frac']:.3f}  edges {r['edges']}")
