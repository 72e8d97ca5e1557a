"""EBNF front end: grammar text -> byte-level expression IR.

Surface semantics follow the reference exactly because they decide mask bits
(SURVEY Appendix A, P7-P12); the implementation is independent:

* literals are UTF-8 of their text; ``\\xHH`` is a raw byte, ``\\uXXXX`` the
  UTF-8 of a code point; simple escapes ``\\n \\t \\r \\" \\\\ \\'``
  (REF grammar.py:290, 326-350, 393-411);
* classes: ``\\] \\- \\^ \\[`` escapes, ``-`` literal first/last, ``]``
  literal only first (REF grammar.py:413-443);
* negated classes must be ASCII/``\\x``-denoted and complement over bytes
  0x00-0xFF (REF grammar.py:576-586);
* positive classes reaching above U+007F become an exact alternation of UTF-8
  byte sequences, surrogates excluded (REF grammar.py:231-281, 565-594);
* ``* + ? {m} {m,} {m,n}``; ``""`` is the empty string (REF grammar.py:445-563);
* root = rule ``root`` else the first rule; undefined references, duplicate
  names, empty grammars and unproductive rules are errors
  (REF grammar.py:629-656); a class matching no byte is an error
  (REF grammar.py:673-678).

IR nodes are small immutable classes; byte sets are 256-bit Python ints.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

__all__ = [
    "GrammarError",
    "Bytes",
    "Lit",
    "Seq",
    "Alt",
    "Rep",
    "Ref",
    "Eps",
    "ParsedGrammar",
    "parse_grammar",
    "utf8_range_sequences",
]

FULL_BYTES = (1 << 256) - 1


class GrammarError(ValueError):
    """Syntax or validation error; carries 1-based line/column when known."""

    def __init__(self, message: str, line: Optional[int] = None, col: Optional[int] = None):
        if line is not None:
            message = f"{message} (line {line}, column {col})"
        super().__init__(message)
        self.line = line
        self.col = col


# -- IR ----------------------------------------------------------------------


@dataclass(frozen=True)
class Bytes:
    mask: int  # bit b set = byte b matches


@dataclass(frozen=True)
class Lit:
    data: bytes


@dataclass(frozen=True)
class Seq:
    items: tuple


@dataclass(frozen=True)
class Alt:
    items: tuple


@dataclass(frozen=True)
class Rep:
    item: object
    lo: int
    hi: Optional[int]


@dataclass(frozen=True)
class Ref:
    name: str


@dataclass(frozen=True)
class Eps:
    pass


@dataclass
class ParsedGrammar:
    names: List[str]  # rule names in source order
    bodies: Dict[str, object]
    root: str


def range_mask(lo: int, hi: int) -> int:
    return ((1 << (hi - lo + 1)) - 1) << lo


# -- UTF-8 lowering of code-point ranges --------------------------------------

_LEN_LIMITS = ((0x00, 0x7F), (0x80, 0x7FF), (0x800, 0xFFFF), (0x10000, 0x10FFFF))


def _cont_split(lo_bytes: bytes, hi_bytes: bytes) -> List[List[Tuple[int, int]]]:
    """Byte-range sequences covering every byte string s with
    lo_bytes <= s <= hi_bytes (same length, all bytes continuation or lead)."""
    n = len(lo_bytes)
    if n == 1:
        return [[(lo_bytes[0], hi_bytes[0])]]
    a, b = lo_bytes[0], hi_bytes[0]
    if a == b:
        return [[(a, a)] + rest for rest in _cont_split(lo_bytes[1:], hi_bytes[1:])]
    out = []
    tail_min, tail_max = bytes([0x80] * (n - 1)), bytes([0xBF] * (n - 1))
    first_full = lo_bytes[1:] == tail_min
    last_full = hi_bytes[1:] == tail_max
    mid_lo = a if first_full else a + 1
    mid_hi = b if last_full else b - 1
    if not first_full:
        out += [[(a, a)] + rest for rest in _cont_split(lo_bytes[1:], tail_max)]
    if mid_lo <= mid_hi:
        out.append([(mid_lo, mid_hi)] + [(0x80, 0xBF)] * (n - 1))
    if not last_full:
        out += [[(b, b)] + rest for rest in _cont_split(tail_min, hi_bytes[1:])]
    return out


def utf8_range_sequences(lo: int, hi: int) -> List[List[Tuple[int, int]]]:
    """Exact UTF-8 byte-range sequences for code points lo..hi (surrogates
    U+D800-DFFF dropped)."""
    pieces = []
    for plo, phi in ((lo, min(hi, 0xD7FF)), (max(lo, 0xE000), hi)):
        if plo > phi:
            continue
        for llo, lhi in _LEN_LIMITS:
            a, b = max(plo, llo), min(phi, lhi)
            if a <= b:
                pieces += _cont_split(chr(a).encode("utf-8"), chr(b).encode("utf-8"))
    return pieces


# -- scanner -----------------------------------------------------------------

_ID0 = frozenset("abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ_")
_ID1 = _ID0 | frozenset("0123456789-")
_HEX = frozenset("0123456789abcdefABCDEF")
_ESC = {"n": 0x0A, "t": 0x09, "r": 0x0D, '"': 0x22, "\\": 0x5C, "'": 0x27}
_PUNCT = {"(": "(", ")": ")", "|": "|", "*": "*", "+": "+", "?": "?"}


class _Scanner:
    """Turns grammar text into (kind, value, line, col) tokens."""

    def __init__(self, text: str):
        self.s = text
        self.i = 0
        self.line = 1
        self.col = 1

    def ch(self, k: int = 0) -> str:
        j = self.i + k
        return self.s[j] if j < len(self.s) else ""

    def bump(self, k: int = 1):
        for _ in range(k):
            if self.i < len(self.s) and self.s[self.i] == "\n":
                self.line, self.col = self.line + 1, 1
            else:
                self.col += 1
            self.i += 1

    def error(self, msg: str):
        raise GrammarError(msg, self.line, self.col)

    def escape(self, in_class: bool) -> Tuple[int, bool]:
        """After a backslash: (value, denotes_raw_byte)."""
        self.bump()
        c = self.ch()
        if not c:
            self.error("unterminated escape")
        if c in _ESC:
            self.bump()
            return _ESC[c], False
        if in_class and c in "]-^[":
            self.bump()
            return ord(c), False
        if c in "xu":
            width = 2 if c == "x" else 4
            digits = self.s[self.i + 1 : self.i + 1 + width]
            if len(digits) != width or not set(digits) <= _HEX:
                self.error(f"\\{c} escape needs {'two' if width == 2 else 'four'} hex digits")
            self.bump(width + 1)
            return int(digits, 16), c == "x"
        self.error(f"unknown escape \\{c}")

    def tokens(self) -> list:
        out = []
        while True:
            c = self.ch()
            if not c:
                out.append(("EOF", None, self.line, self.col))
                return out
            if c in " \t\r\n":
                self.bump()
            elif c == "#":
                while self.ch() not in ("", "\n"):
                    self.bump()
            elif c in _ID0:
                line, col, j = self.line, self.col, self.i
                while self.ch() in _ID1 and self.ch():
                    self.bump()
                out.append(("IDENT", self.s[j : self.i], line, col))
            elif c == ":" and self.s.startswith("::=", self.i):
                out.append(("DEFINE", None, self.line, self.col))
                self.bump(3)
            elif c == '"':
                out.append(self.literal())
            elif c == "[":
                out.append(self.char_class())
            elif c in _PUNCT:
                out.append((_PUNCT[c], None, self.line, self.col))
                self.bump()
            elif c == "{":
                out.append(self.bounds())
            else:
                self.error(f"unexpected character {c!r}")

    def literal(self):
        line, col = self.line, self.col
        self.bump()
        buf = bytearray()
        while True:
            c = self.ch()
            if c in ("", "\n"):
                raise GrammarError("unterminated string literal", line, col)
            if c == '"':
                self.bump()
                return ("LIT", bytes(buf), line, col)
            if c == "\\":
                v, raw = self.escape(in_class=False)
                if raw:
                    buf.append(v)
                else:
                    try:
                        buf += chr(v).encode("utf-8")
                    except UnicodeEncodeError:
                        raise GrammarError(f"escape \\u{v:04X} is a lone surrogate", line, col) from None
            else:
                buf += c.encode("utf-8")
                self.bump()

    def char_class(self):
        line, col = self.line, self.col
        self.bump()
        negated = self.ch() == "^"
        if negated:
            self.bump()
        members = []  # (lo, hi, raw_byte)
        while True:
            c = self.ch()
            if c in ("", "\n"):
                raise GrammarError("unterminated character class", line, col)
            if c == "]" and members:
                self.bump()
                return ("CLASS", (members, negated), line, col)
            lo, lo_raw = self.class_atom()
            hi, hi_raw = lo, lo_raw
            if self.ch() == "-" and self.ch(1) not in ("]", ""):
                self.bump()
                hi, hi_raw = self.class_atom()
            if hi < lo:
                raise GrammarError(f"class range out of order: {lo:#x}-{hi:#x}", line, col)
            members.append((lo, hi, lo_raw or hi_raw))

    def class_atom(self) -> Tuple[int, bool]:
        c = self.ch()
        if c == "\\":
            return self.escape(in_class=True)
        self.bump()
        return ord(c), False

    def bounds(self):
        line, col = self.line, self.col
        self.bump()

        def number() -> str:
            d = ""
            while self.ch().isdigit():
                d += self.ch()
                self.bump()
            return d

        lo_s = number()
        if not lo_s:
            self.error("repeat bounds need a count")
        lo = int(lo_s)
        hi: Optional[int] = lo
        if self.ch() == ",":
            self.bump()
            hi_s = number()
            hi = int(hi_s) if hi_s else None
        if self.ch() != "}":
            self.error("unterminated repeat bounds")
        self.bump()
        return ("BOUNDS", (lo, hi), line, col)


# -- parser ------------------------------------------------------------------


def _lower_class(members, negated, line, col):
    byte_mask = 0
    cps = []
    for lo, hi, raw in members:
        if raw or hi <= 0x7F:
            if hi > 0xFF:
                raise GrammarError(f"byte escape out of range: {hi:#x}", line, col)
            byte_mask |= range_mask(lo, hi)
        else:
            cps.append((lo, hi))
    if negated:
        if cps:
            raise GrammarError("negated classes may only contain ASCII or \\xHH members", line, col)
        return Bytes(FULL_BYTES & ~byte_mask)
    if not cps:
        return Bytes(byte_mask)
    alts = []
    cp_ascii = 0
    for lo, hi in cps:
        if hi > 0x10FFFF:
            raise GrammarError(f"code point out of range: {hi:#x}")
        if lo <= 0x7F:
            cp_ascii |= range_mask(lo, 0x7F)
            lo = 0x80
        for seq in utf8_range_sequences(lo, hi):
            parts = tuple(Bytes(range_mask(a, b)) for a, b in seq)
            alts.append(parts[0] if len(parts) == 1 else Seq(parts))
    if not alts and not cp_ascii:  # e.g. only surrogates (REF grammar.py:277-278)
        raise GrammarError("empty character class after lowering")
    if byte_mask | cp_ascii:
        alts.insert(0, Bytes(byte_mask | cp_ascii))
    return alts[0] if len(alts) == 1 else Alt(tuple(alts))


class _Parser:
    def __init__(self, toks):
        self.t = toks
        self.k = 0

    def peek(self, off: int = 0):
        return self.t[min(self.k + off, len(self.t) - 1)]

    def take(self):
        tok = self.t[self.k]
        if tok[0] != "EOF":
            self.k += 1
        return tok

    def expect(self, kind: str):
        tok = self.take()
        if tok[0] != kind:
            raise GrammarError(f"expected {_KIND_NAMES.get(kind, kind)}, got {_KIND_NAMES.get(tok[0], tok[0])}", tok[2], tok[3])
        return tok

    def rules(self):
        out = []
        while self.peek()[0] != "EOF":
            name = self.expect("IDENT")
            self.expect("DEFINE")
            out.append((name[1], self.alternation(), name[2], name[3]))
        return out

    def alternation(self):
        alts = [self.sequence()]
        while self.peek()[0] == "|":
            self.take()
            alts.append(self.sequence())
        return alts[0] if len(alts) == 1 else Alt(tuple(alts))

    def sequence(self):
        items = []
        while True:
            kind = self.peek()[0]
            if kind in ("|", ")", "EOF") or (kind == "IDENT" and self.peek(1)[0] == "DEFINE"):
                break
            items.append(self.postfix())
        if not items:
            return Eps()
        return items[0] if len(items) == 1 else Seq(tuple(items))

    def postfix(self):
        e = self.atom()
        while True:
            kind, val, line, col = self.peek()
            if kind == "*":
                e = Rep(e, 0, None)
            elif kind == "+":
                e = Rep(e, 1, None)
            elif kind == "?":
                e = Rep(e, 0, 1)
            elif kind == "BOUNDS":
                lo, hi = val
                if hi is not None and hi < lo:
                    raise GrammarError(f"bad repeat bounds {{{lo},{hi}}}", line, col)
                e = Rep(e, lo, hi)
            else:
                return e
            self.take()

    def atom(self):
        kind, val, line, col = self.take()
        if kind == "LIT":
            return Lit(val) if val else Eps()
        if kind == "CLASS":
            return _lower_class(val[0], val[1], line, col)
        if kind == "IDENT":
            return Ref(val)
        if kind == "(":
            e = self.alternation()
            self.expect(")")
            return e
        raise GrammarError(f"unexpected {_KIND_NAMES.get(kind, kind)} in expression", line, col)


_KIND_NAMES = {"(": "LPAREN", ")": "RPAREN", "|": "PIPE", "*": "STAR", "+": "PLUS", "?": "QMARK", "LIT": "LITERAL"}


def _walk(e):
    yield e
    if isinstance(e, (Seq, Alt)):
        for x in e.items:
            yield from _walk(x)
    elif isinstance(e, Rep):
        yield from _walk(e.item)


def _derives(e, productive: set) -> bool:
    if isinstance(e, Bytes):
        return e.mask != 0
    if isinstance(e, (Lit, Eps)):
        return True
    if isinstance(e, Seq):
        return all(_derives(x, productive) for x in e.items)
    if isinstance(e, Alt):
        return any(_derives(x, productive) for x in e.items)
    if isinstance(e, Rep):
        return e.lo == 0 or _derives(e.item, productive)
    return e.name in productive


def parse_grammar(text: str, root_rule_name: Optional[str] = None) -> ParsedGrammar:
    """Parse and validate grammar text (REF grammar.py:629-666 semantics).

    ``root_rule_name`` (XGrammar's compile_grammar kwarg) overrides the
    default root choice when given."""
    raw = _Parser(_Scanner(text).tokens()).rules()
    if not raw:
        raise GrammarError("empty grammar")
    bodies: Dict[str, object] = {}
    for name, body, line, col in raw:
        if name in bodies:
            raise GrammarError(f"duplicate rule name {name!r}", line, col)
        bodies[name] = body
    for name, body, line, col in raw:
        for e in _walk(body):
            if isinstance(e, Ref) and e.name not in bodies:
                raise GrammarError(f"undefined rule reference {e.name!r} in {name!r}", line, col)
    productive: set = set()
    grew = True
    while grew:
        grew = False
        for name, body, _, _ in raw:
            if name not in productive and _derives(body, productive):
                productive.add(name)
                grew = True
    dead = [name for name, _, _, _ in raw if name not in productive]
    if dead:
        raise GrammarError(f"rules derive no strings (empty language): {', '.join(dead)}")
    for name, body, _, _ in raw:
        if any(isinstance(e, Bytes) and e.mask == 0 for e in _walk(body)):
            raise GrammarError("character class matches no byte")
    names = [r[0] for r in raw]
    if root_rule_name is not None:
        if root_rule_name not in bodies:
            raise GrammarError(f"root rule {root_rule_name!r} is not defined")
        root = root_rule_name
    else:
        root = "root" if "root" in bodies else names[0]
    return ParsedGrammar(names, bodies, root)
