"""XGrammar-compatible compile API (names and kwargs of xgrammar 0.2.0,
xgrammar/tokenizer_info.py:69-104, xgrammar/compiler.py:100-327).

Behaviour follows the reference grammask wherever the two differ (SURVEY
§0.3): byte-level negated classes, explicit special tokens that are never
allowed, a single EOS.  ``TokenizerInfo`` therefore takes an extra
``special_token_ids`` argument; the stop token must be one id (the first of
``stop_token_ids``).
"""

from __future__ import annotations

import enum
import json
import threading
from typing import Dict, List, Optional, Sequence, Union

import torch

from .automaton import AutomatonOptions
from .engine import CompiledDeviceGrammar, DeviceVocab, compile_on_device
from .schema import schema_to_grammar_text
from .vocab import BYTE_LEVEL_DECODE, Vocabulary, vocab_from_tokens

__all__ = ["VocabType", "TokenizerInfo", "GrammarCompiler", "CompiledGrammar", "BUILTIN_JSON_GRAMMAR"]

# ECMA-404 JSON, the grammar behind compile_builtin_json_grammar (the
# reference's JSON_ECMA404 workload, REF grammars.py:15-35, restated).
BUILTIN_JSON_GRAMMAR = r'''
root     ::= element
element  ::= ws value ws
value    ::= object | array | string | number | "true" | "false" | "null"
object   ::= "{" ws "}" | "{" members "}"
members  ::= member ("," member)*
member   ::= ws string ws ":" element
array    ::= "[" ws "]" | "[" elements "]"
elements ::= element ("," element)*
string   ::= "\"" char* "\""
char     ::= [^"\\\x00-\x1F] | "\\" escape
escape   ::= [\"\\/bfnrt] | "u" hex hex hex hex
hex      ::= [0-9a-fA-F]
number   ::= integer fraction exponent
integer  ::= "-"? ("0" | onenine digit*)
digit    ::= [0-9]
onenine  ::= [1-9]
fraction ::= ("." digit+)?
exponent ::= (("e" | "E") ("+" | "-")? digit+)?
ws       ::= [ \t\n\r]*
'''


class VocabType(enum.Enum):
    RAW = 0
    BYTE_FALLBACK = 1
    BYTE_LEVEL = 2


def _decode_token(tok: Union[str, bytes], vocab_type: VocabType) -> bytes:
    if isinstance(tok, bytes):
        return tok
    if vocab_type == VocabType.BYTE_LEVEL:
        try:
            return bytes(BYTE_LEVEL_DECODE[c] for c in tok)
        except KeyError:
            return tok.encode("utf-8")
    if vocab_type == VocabType.BYTE_FALLBACK:
        if len(tok) == 6 and tok.startswith("<0x") and tok.endswith(">"):
            try:
                return bytes([int(tok[3:5], 16)])
            except ValueError:
                pass
        return tok.replace("▁", " ").encode("utf-8")
    return tok.encode("utf-8")


class TokenizerInfo:
    """Vocabulary + special/stop tokens, resident on the current CUDA device."""

    def __init__(
        self,
        encoded_vocab: Union[Sequence[bytes], Sequence[str]],
        vocab_type: VocabType = VocabType.RAW,
        *,
        vocab_size: Optional[int] = None,
        stop_token_ids: Optional[Union[List[int], int]] = None,
        add_prefix_space: bool = False,
        special_token_ids: Optional[Sequence[int]] = None,
    ) -> None:
        toks = [_decode_token(t, vocab_type) for t in encoded_vocab]
        if vocab_size is not None:
            if vocab_size < len(toks):
                raise ValueError("vocab_size is smaller than the encoded vocabulary")
            toks += [b""] * (vocab_size - len(toks))  # padding ids: empty => never allowed
        if isinstance(stop_token_ids, int):
            stop_token_ids = [stop_token_ids]
        if not stop_token_ids:
            raise ValueError("stop_token_ids is required (grammask semantics: exactly one EOS)")
        eos = int(stop_token_ids[0])
        specials = set(int(s) for s in (special_token_ids or ())) | set(int(s) for s in stop_token_ids)
        self._init(vocab_from_tokens(toks, eos, sorted(specials)), vocab_type, add_prefix_space)

    def _init(self, vocab: Vocabulary, vocab_type: VocabType, add_prefix_space: bool):
        self.vocab = vocab
        self.vocab_type = vocab_type
        self.add_prefix_space = add_prefix_space
        self.device_vocab = DeviceVocab(vocab)

    @classmethod
    def from_vocabulary(cls, vocab: Vocabulary) -> "TokenizerInfo":
        self = cls.__new__(cls)
        self._init(vocab, VocabType.RAW, False)
        return self

    @property
    def vocab_size(self) -> int:
        return self.vocab.size

    @property
    def stop_token_ids(self) -> List[int]:
        return [self.vocab.eos_id]

    @property
    def special_token_ids(self) -> List[int]:
        return sorted(self.vocab.special_tokens)

    @property
    def decoded_vocab(self) -> List[bytes]:
        return list(self.vocab.tokens)


class CompiledGrammar:
    """Automaton tables + device cache for one grammar and tokenizer."""

    def __init__(self, dev: CompiledDeviceGrammar, tokenizer_info: TokenizerInfo, grammar_text: str):
        self._dev = dev
        self.tokenizer_info = tokenizer_info
        self.grammar_text = grammar_text

    @property
    def memory_size_bytes(self) -> int:
        return int(self._dev.cache.stats["row_bytes"]) + 4 * int(self._dev.cache.stats["dependent_total"])

    @property
    def stats(self) -> dict:
        return dict(self._dev.stats)

    @property
    def compile_ms(self) -> dict:
        return dict(self._dev.timings_ms)


class GrammarCompiler:
    """Compiles grammars into CompiledGrammar; caches by grammar text."""

    def __init__(
        self,
        tokenizer_info: TokenizerInfo,
        *,
        max_threads: int = 8,
        cache_enabled: bool = True,
        cache_limit_bytes: int = -1,
        options: Optional[AutomatonOptions] = None,
        group=None,
    ) -> None:
        self._threads = max(1, int(max_threads)) if isinstance(max_threads, int) else 8  # batch compiles
        self.tokenizer_info = tokenizer_info
        self._cache_enabled = cache_enabled
        self._cache_limit = cache_limit_bytes
        self._options = options
        self._group = group
        self._memo: Dict[tuple, CompiledGrammar] = {}
        self._lock = threading.Lock()

    def _compile(self, text: str, root_rule_name: Optional[str] = None, parsed=None) -> CompiledGrammar:
        key = (text, root_rule_name)
        if self._cache_enabled:
            with self._lock:
                hit = self._memo.get(key)
            if hit is not None:
                return hit
        dev = compile_on_device(text, self.tokenizer_info.device_vocab, self._options,
                                root_rule_name=root_rule_name, group=self._group, parsed=parsed)
        cg = CompiledGrammar(dev, self.tokenizer_info, text)
        if self._cache_enabled:
            with self._lock:
                self._memo[key] = cg
                if self._cache_limit >= 0:
                    while self._memo and sum(c.memory_size_bytes for c in self._memo.values()) > self._cache_limit:
                        self._memo.pop(next(iter(self._memo)))
        return cg

    def compile_grammar(self, grammar: str, *, root_rule_name: str = "root") -> CompiledGrammar:
        """EBNF text -> CompiledGrammar.  The root is ``root_rule_name`` if that
        rule exists, else the grammask default (first rule)."""
        import dataclasses

        from .automaton import parse_grammar_native

        g = parse_grammar_native(grammar)  # parsed once (native): the root is chosen on the result
        root = root_rule_name if root_rule_name in g.names else None
        if root is not None and g.root != root:
            g = dataclasses.replace(g, root=root)
        return self._compile(grammar, root, parsed=g)

    def compile_json_schema(
        self,
        schema: Union[str, dict],
        *,
        any_whitespace: bool = True,
        indent: Optional[int] = None,
        separators=None,
        strict_mode: bool = True,
        max_whitespace_cnt: Optional[int] = None,
    ) -> CompiledGrammar:
        """JSON Schema (grammask subset, REF schema.py:25-35) -> CompiledGrammar.
        ``any_whitespace=False`` selects the reference's strict mode; the
        formatting kwargs are accepted and ignored (the reference fixes one
        spelling)."""
        del indent, separators, strict_mode, max_whitespace_cnt
        if isinstance(schema, dict):
            schema = json.dumps(schema)
        return self._compile(schema_to_grammar_text(schema, whitespace=any_whitespace))

    def compile_json_schemas(self, schemas, *, any_whitespace: bool = True, max_workers: Optional[int] = None):
        """Compile many JSON schemas (e.g. BASELINE config 5: one per request)
        on ``max_workers`` host threads (default: the compiler's
        ``max_threads``): the native front end and the device build release
        the GIL, so schemas overlap; results in input order."""
        from concurrent.futures import ThreadPoolExecutor

        n = max_workers or self._threads
        if n <= 1 or len(schemas) <= 1:
            return [self.compile_json_schema(s, any_whitespace=any_whitespace) for s in schemas]
        dev = torch.cuda.current_device()

        def one(sch):
            torch.cuda.set_device(dev)
            return self.compile_json_schema(sch, any_whitespace=any_whitespace)

        with ThreadPoolExecutor(max_workers=n) as ex:
            return list(ex.map(one, schemas))

    def compile_builtin_json_grammar(self) -> CompiledGrammar:
        return self._compile(BUILTIN_JSON_GRAMMAR)

    def clear_cache(self) -> None:
        with self._lock:
            self._memo.clear()
