"""Reader for tests/golden/*.kbt fixtures (hand-worked tiny ABoxes).

Format (after SPEC.md:120-129's KB text format, restricted to what the
fixtures need):
  ; comment lines (each fixture cites its source passage)
  #individuals      names separated by whitespace
  #concepts / #roles / #numeric-roles   names
  #concept-assertions   <concept> <individual>
  #role-assertions      <role> <subject> <object>
  #numeric-assertions   <numeric-role> <subject> <decimal>
  #string-roles         names
  #string-assertions    <string-role> <subject> "<literal>"   (\" escapes a quote)
  #examples             + <individual> | - <individual>
  #flags                compat_paper_max
  #hypotheses           <s-expr> => {i1, i2, ...} [tp fp fn tn]
"""
import math
import os
import re

import numpy as np

from synth.format import COMPILE_COMPAT_PAPER_MAX, kb_from_sets, parse

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(path):
    sec = None
    ind, con, rol, num, srl = [], [], [], [], []
    ca, ra, na, sa, ex, hy = [], [], [], [], [], []
    flags = 0
    for raw in open(path):
        line = raw.strip()
        if not line or line.startswith(";"):
            continue
        if line.startswith("#"):
            sec = line[1:]
            continue
        if sec == "individuals":
            ind += line.split()
        elif sec == "concepts":
            con += line.split()
        elif sec == "roles":
            rol += line.split()
        elif sec == "numeric-roles":
            num += line.split()
        elif sec == "string-roles":
            srl += line.split()
        elif sec == "string-assertions":
            m = re.match(r'(\S+)\s+(\S+)\s+"((?:[^"\\]|\\.)*)"$', line)
            assert m, line
            sa.append((m.group(1), m.group(2), m.group(3).replace('\\"', '"').replace("\\\\", "\\")))
        elif sec == "concept-assertions":
            ca.append(line.split())
        elif sec == "role-assertions":
            ra.append(line.split())
        elif sec == "numeric-assertions":
            na.append(line.split())
        elif sec == "examples":
            ex.append(line.split())
        elif sec == "flags":
            if "compat_paper_max" in line:
                flags |= COMPILE_COMPAT_PAPER_MAX
        elif sec == "hypotheses":
            hy.append(line)
    ii = {s: i for i, s in enumerate(ind)}
    concepts = [[] for _ in con]
    for c, a in ca:
        concepts[con.index(c)].append(ii[a])
    roles = [[] for _ in rol]
    for r, s, o in ra:
        roles[rol.index(r)].append((ii[s], ii[o]))
    data = [[] for _ in num]
    for d, s, v in na:
        data[num.index(d)].append((ii[s], float(np.float32(float(v)))))
    pos = [ii[a] for s, a in ex if s == "+"]
    neg = [ii[a] for s, a in ex if s == "-"]
    strings = [[] for _ in srl]
    for r, s_, v in sa:
        strings[srl.index(r)].append((ii[s_], v.encode()))
    kb = kb_from_sets(len(ind), concepts, roles, data, pos, neg, strings)
    names = {"concepts": con, "roles": rol, "data": num, "strings": srl}
    cases = []
    for line in hy:
        m = re.match(r"(.*)=>\s*\{([^}]*)\}\s*(.*)$", line)
        assert m, line
        tree = parse(m.group(1), names)
        members = {ii[s.strip()] for s in m.group(2).split(",") if s.strip()}
        counts = tuple(int(x) for x in m.group(3).split()) if m.group(3).strip() else None
        cases.append((m.group(1).strip(), tree, members, counts))
    return kb, cases, flags


def all_fixtures():
    return sorted(os.path.join(GOLDEN, f) for f in os.listdir(GOLDEN) if f.endswith(".kbt"))


def load_names(path):
    """The fixture's declared names per kind (hedl_compile_text's name table)."""
    sec, names = None, {"concepts": [], "roles": [], "data": [], "strings": []}
    key = {"concepts": "concepts", "roles": "roles", "numeric-roles": "data", "string-roles": "strings"}
    for raw in open(path):
        line = raw.strip()
        if not line or line.startswith(";"):
            continue
        if line.startswith("#"):
            sec = line[1:]
            continue
        if sec in key:
            names[key[sec]] += line.split()
    return names
