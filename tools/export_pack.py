"""Export the reference's ModelPack for the benchmark fluid to JSON.

Run once in a container that has /root/reference (the GPU box does not):
    python tools/export_pack.py
It writes paper_1811_11992_b200/data/tube3_pack.json from the reference's own
``build_pack`` (assembly.py:83-172) applied to the C2 deck, so that our side
uses exactly the reference's flattened constants.
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tools.refdeck import reference_simulator  # noqa: E402
from paper_1811_11992_b200 import configs  # noqa: E402
from paper_1811_11992_b200.model import DATA_DIR, pack_to_dict  # noqa: E402


def main():
    sim = reference_simulator(configs.config("small3d"))
    d = pack_to_dict(sim.pack)
    d["source"] = ("reference iscsim build_pack on tube.deck fluid minus the "
                   "light-oil oxidation reaction (tools/export_pack.py)")
    os.makedirs(DATA_DIR, exist_ok=True)
    path = os.path.join(DATA_DIR, "tube3_pack.json")
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(d, fh, indent=1)
    print("wrote", path, "nreac", len(d["law_codes"]["data"]))


if __name__ == "__main__":
    main()
