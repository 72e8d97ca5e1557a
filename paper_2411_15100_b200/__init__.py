"""B200-native token-mask engine: XGrammar's hot path (arXiv 2411.15100).

XGrammar-compatible API: TokenizerInfo, GrammarCompiler, CompiledGrammar,
GrammarMatcher, BatchGrammarMatcher, allocate_token_bitmask,
apply_token_bitmask_inplace.  The reference's own (grammask) API lives in
``paper_2411_15100_b200.compat``.
"""

from .bitmask import (
    allocate_token_bitmask,
    apply_token_bitmask_inplace,
    bitmask_dtype,
    get_bitmask_shape,
    reset_token_bitmask,
)
from .automaton import AutomatonOptions, StateLimitError
from .compiler import BUILTIN_JSON_GRAMMAR, CompiledGrammar, GrammarCompiler, TokenizerInfo, VocabType
from .engine import MatcherError
from .grammar import GrammarError
from .matcher import BatchGrammarMatcher, GrammarMatcher, batch_accept, batch_fill
from .schema import SchemaError
from .vocab import Vocabulary, load_vocab, loads_vocab, synth_vocab, vocab_from_tokens

__version__ = "0.1.0"
