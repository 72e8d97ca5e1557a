"""JSON Schema subset -> grammar text (behind compile_json_schema).

The accepted language follows REF schema.py exactly: keywords
type / properties / required / additionalProperties:false / items /
minItems / maxItems / enum / const (REF schema.py:25-35); ECMA-404 lexical
rules for strings and numbers (REF schema.py:72-84); required properties in
schema order, then optional ones, each independently present, fixed order
(REF schema.py:170-205); arrays with bounds (REF schema.py:207-228);
whitespace ``[ \\t\\n\\r]*`` between tokens unless strict
(REF schema.py:231-246).
"""

from __future__ import annotations

import json
from typing import Dict, List, Union

__all__ = ["SchemaError", "schema_to_grammar_text"]

_KEYWORDS = frozenset(
    ["type", "properties", "required", "additionalProperties", "items", "enum", "const", "minItems", "maxItems"]
)
_SCALAR_TYPES = {
    "string": "jstring",
    "number": "jnumber",
    "integer": "jinteger",
    "boolean": "jboolean",
    "null": "jnull",
}
_LIBRARY = {
    "jstring": ('"\\"" jchar* "\\""', ["jchar"]),
    "jchar": ('[^"\\\\\\x00-\\x1F] | "\\\\" jescape', ["jescape"]),
    "jescape": ('[\\"\\\\/bfnrt] | "u" jhex jhex jhex jhex', ["jhex"]),
    "jhex": ("[0-9a-fA-F]", []),
    "jinteger": ('"-"? ("0" | [1-9] [0-9]*)', []),
    "jnumber": ("jinteger jfraction jexponent", ["jinteger", "jfraction", "jexponent"]),
    "jfraction": ('("." [0-9]+)?', []),
    "jexponent": ("([eE] [-+]? [0-9]+)?", []),
    "jboolean": ('"true" | "false"', []),
    "jnull": ('"null"', []),
    "ws": ("[ \\t\\n\\r]*", []),
}


class SchemaError(ValueError):
    """Schema outside the supported subset (names the offending keywords)."""

    def __init__(self, message: str, unsupported=()):
        if unsupported:
            message = f"{message}: {', '.join(sorted(unsupported))}"
        super().__init__(message)
        self.unsupported = tuple(sorted(unsupported))


def _quote(text: str) -> str:
    """Grammar literal for the UTF-8 bytes of ``text``."""
    out = []
    for b in text.encode("utf-8"):
        if b in (0x22, 0x5C):
            out.append("\\" + chr(b))
        elif b in (0x0A, 0x09, 0x0D):
            out.append({0x0A: "\\n", 0x09: "\\t", 0x0D: "\\r"}[b])
        elif 0x20 <= b <= 0x7E:
            out.append(chr(b))
        else:
            out.append(f"\\x{b:02X}")
    return '"' + "".join(out) + '"'


class _Lowering:
    def __init__(self, whitespace: bool):
        self.ws = " ws " if whitespace else ""
        self.defs: Dict[str, str] = {}
        self.n = 0

    def lib(self, name: str) -> str:
        if name not in self.defs:
            body, deps = _LIBRARY[name]
            self.defs[name] = body
            for d in deps:
                self.lib(d)
        return name

    def fresh(self) -> str:
        self.n += 1
        return f"v{self.n}"

    @staticmethod
    def scalar(value) -> str:
        if isinstance(value, (dict, list)):
            raise SchemaError("enum/const values must be scalars")
        return _quote(json.dumps(value))

    def node(self, s) -> str:
        if not isinstance(s, dict):
            raise SchemaError("schema nodes must be objects")
        bad = set(s) - _KEYWORDS
        if bad:
            raise SchemaError("unsupported schema keywords", bad)
        name = self.fresh()
        if self.ws:
            self.lib("ws")
        if "const" in s:
            self.defs[name] = self.scalar(s["const"])
        elif "enum" in s:
            vals = s["enum"]
            if not isinstance(vals, list) or not vals:
                raise SchemaError("enum must be a non-empty array")
            self.defs[name] = " | ".join(self.scalar(v) for v in vals)
        else:
            t = s.get("type")
            if t is None:
                raise SchemaError("schema node needs one of: type, enum, const")
            if isinstance(t, list):
                raise SchemaError("unsupported schema keywords", {"type (as a list)"})
            if t in _SCALAR_TYPES:
                self.defs[name] = self.lib(_SCALAR_TYPES[t])
            elif t == "object":
                self.defs[name] = None  # reserve the position (rule order is cosmetic)
                self.defs[name] = self.obj(s)
            elif t == "array":
                self.defs[name] = None
                self.defs[name] = self.arr(s)
            else:
                raise SchemaError(f"unsupported type {t!r}")
        return name

    def obj(self, s) -> str:
        if s.get("additionalProperties") is not False:
            raise SchemaError("objects require additionalProperties: false (free-form objects are unsupported)")
        props = s.get("properties", {})
        if not isinstance(props, dict):
            raise SchemaError("properties must be an object")
        req = s.get("required", [])
        if not isinstance(req, list) or any(r not in props for r in req):
            raise SchemaError("required must list property names present in properties")
        ws = self.ws
        comma = f'{ws}","{ws}'
        members = [(k in req, f'{_quote(json.dumps(k))}{ws}":"{ws}{self.node(v)}') for k, v in props.items()]
        required = [m for r, m in members if r]
        optional = [m for r, m in members if not r]
        tail = lambda ms: "".join(f"({comma}{m})?" for m in ms)  # noqa: E731
        if required:
            body = comma.join(required) + tail(optional)
        elif optional:
            body = "( " + " | ".join(optional[i] + tail(optional[i + 1 :]) for i in range(len(optional))) + " )?"
        else:
            body = ""
        return f'"{{"{ws}{body}{ws}"}}"' if body else f'"{{"{ws}"}}"'

    def arr(self, s) -> str:
        if s.get("items") is None:
            raise SchemaError("arrays require items")
        lo, hi = s.get("minItems", 0), s.get("maxItems")
        if not isinstance(lo, int) or lo < 0 or (hi is not None and (not isinstance(hi, int) or hi < lo)):
            raise SchemaError("bad minItems/maxItems")
        item = self.node(s["items"])
        ws = self.ws
        if hi == 0:
            return f'"["{ws}"]"'
        if hi is None:
            rep = "*" if lo == 0 else f"{{{lo - 1},}}"
        else:
            rep = f"{{{max(lo - 1, 0)},{hi - 1}}}"
        seq = f'{item} ({ws}","{ws}{item}){rep}'
        return f'"["{ws}( {seq} )?{ws}"]"' if lo == 0 else f'"["{ws}{seq}{ws}"]"'


def schema_to_grammar_text(schema: Union[str, dict], *, whitespace: bool = True) -> str:
    """Grammar text whose language is the schema's JSON documents."""
    if isinstance(schema, str):
        try:
            schema = json.loads(schema)
        except json.JSONDecodeError as exc:
            raise SchemaError(f"schema is not valid JSON: {exc}") from exc
    low = _Lowering(whitespace)
    body = low.node(schema)
    ws = "ws " if whitespace else ""
    lines: List[str] = [f"root ::= {ws}{body} {ws}".rstrip()]
    lines += [f"{k} ::= {v}" for k, v in low.defs.items()]
    return "\n".join(lines) + "\n"
