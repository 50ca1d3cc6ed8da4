"""Exact, single-occurrence source edits for scripted refactors: sedit(path, [(old, new), ...])."""


def sedit(path, pairs):
    s = open(path).read()
    for old, new in pairs:
        n = s.count(old)
        if n != 1:
            raise SystemExit(f"{path}: expected exactly one occurrence, found {n}: {old[:80]!r}")
        s = s.replace(old, new)
    open(path, "w").write(s)
