"""Minimal unifdef: fold preprocessor conditionals on macros with known values.

    python tools/unifdef.py FILE -DNAME=VALUE ...      (rewrites FILE in place)

Handles #if / #ifdef / #ifndef / #elif / #else / #endif whose expression uses only the
given macros (plus integer literals, !, &&, ||, ==, !=, <, >, <=, >=); conditionals that
mention anything else are left untouched.  The '#ifndef NAME / #define NAME v / #endif'
default blocks of the given macros are removed, and remaining uses of NAME in code are
replaced by its value.  Used once to delete the round-1 experiment switches."""
import re
import sys


def evaluate(expr, defs):
    expr = re.sub(r"//.*", "", expr)
    names = set(re.findall(r"[A-Za-z_]\w*", expr)) - {"defined"}
    if not names <= set(defs):
        return None
    e = re.sub(r"defined\s*\(?\s*(\w+)\s*\)?", lambda m: "1", expr)
    for n in sorted(names, key=len, reverse=True):
        e = re.sub(rf"\b{n}\b", str(defs[n]), e)
    e = e.replace("&&", " and ").replace("||", " or ").replace("!=", " ne ")
    e = re.sub(r"!(?!=)", " not ", e).replace(" ne ", "!=")
    e = re.sub(r"//.*", "", e)
    return bool(eval(e))


def process(lines, defs):
    out = []
    stack = []  # per #if: [mode, taken] ; mode: 'keep' (unknown), 'fold'
    emitting = lambda: all(s[2] for s in stack if s[0] == "fold")
    i = 0
    while i < len(lines):
        ln = lines[i]
        m = re.match(r"\s*#\s*(if|ifdef|ifndef|elif|else|endif)\b(.*)", ln)
        if m:
            kw, rest = m.group(1), m.group(2).strip()
            if kw in ("if", "ifdef", "ifndef"):
                if kw == "ifdef":
                    val = True if rest.split()[0] in defs else None
                elif kw == "ifndef":
                    name = rest.split()[0]
                    if name in defs:  # default-value block of a folded macro: drop it whole
                        depth = 1
                        j = i + 1
                        while depth:
                            if re.match(r"\s*#\s*if", lines[j]):
                                depth += 1
                            elif re.match(r"\s*#\s*endif", lines[j]):
                                depth -= 1
                            j += 1
                        i = j
                        continue
                    val = None
                else:
                    val = evaluate(rest, defs)
                if val is None:
                    stack.append(["keep", None, True])
                    if emitting():
                        out.append(ln)
                else:
                    stack.append(["fold", val, val])
            elif kw == "elif":
                top = stack[-1]
                if top[0] == "keep":
                    if emitting():
                        out.append(ln)
                else:
                    val = evaluate(rest, defs)
                    if val is None:
                        raise SystemExit(f"cannot fold #elif {rest}")
                    top[2] = (not top[1]) and val
                    top[1] = top[1] or val
            elif kw == "else":
                top = stack[-1]
                if top[0] == "keep":
                    if emitting():
                        out.append(ln)
                else:
                    top[2] = not top[1]
            else:  # endif
                top = stack.pop()
                if top[0] == "keep" and emitting():
                    out.append(ln)
            i += 1
            continue
        if emitting():
            for n, v in defs.items():
                ln = re.sub(rf"\b{n}\b", str(v), ln)
            out.append(ln)
        i += 1
    return out


if __name__ == "__main__":
    path = sys.argv[1]
    defs = {}
    for a in sys.argv[2:]:
        k, v = a[2:].split("=")
        defs[k] = int(v)
    with open(path) as fh:
        lines = fh.readlines()
    with open(path, "w") as fh:
        fh.writelines(process(lines, defs))
