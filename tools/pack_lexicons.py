"""Pack the reference's router lexicons into one data file for the package.

    python tools/pack_lexicons.py          # build container only (reads /root/reference)

The lexicons are contract data, not code: cascadesim's router
(pkg/src/cascadesim/router.py:58-87) reads six small text files under
data/lexicons/ and every hardness value depends on them.  This script stores
their non-empty stripped lines -- exactly what ``router._read_lines`` returns
(router.py:58-61) -- in ``paper_2509_00642_b200/data/lexicons.json`` so the
GPU text path can run where the reference is not installed.
"""

import json
import os
import sys

SRC = "/root/reference/pkg/src/cascadesim/data/lexicons"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2509_00642_b200",
                   "data", "lexicons.json")
NAMES = ("word_frequency.tsv", "abstract_nouns.txt", "action_verbs.txt", "adjectives.txt",
         "noun_markers.txt", "spatial_phrases.txt")


def main():
    doc = {"source": "cascadesim 0.1.0 pkg/src/cascadesim/data/lexicons (router._read_lines)",
           "files": {}}
    for name in NAMES:
        with open(os.path.join(SRC, name), encoding="utf-8") as fh:
            text = fh.read()
        doc["files"][name] = [line.strip() for line in text.splitlines() if line.strip()]
    with open(OUT, "w", encoding="utf-8") as fh:
        json.dump(doc, fh, indent=0, sort_keys=True)
        fh.write("\n")
    print({k: len(v) for k, v in doc["files"].items()}, file=sys.stderr)


if __name__ == "__main__":
    main()
