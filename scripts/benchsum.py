"""One-line summaries of bench JSON lines (helper for the evidence passes)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads([ln for ln in open(f) if ln.lstrip().startswith("{")][-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    c = d.get("codec") or {}
    fm = c.get("family_model", {})
    print(f, d.get("value"), d.get("unit"), "frac", (d.get("roofline") or {}).get("frac"),
          "e2e", (d.get("e2e") or {}).get("value"), "enc_dev", fm.get("encode_device_frac"),
          "dec", fm.get("decode_frac"), "dec_ms", c.get("decode_ms_per_family"),
          "sel", (d.get("selection") or {}).get("frac"), "clk", d.get("clocks"))
