"""Textual chain specifications.

Same grammar, stage catalog and errors as the reference's
``wavepipe.chainspec`` (pkg/src/wavepipe/chainspec.py:1-250)::

    chain  := stage ("|" stage)*
    stage  := name "(" [arg ("," arg)*] ")"
    arg    := value | name "=" value
    value  := number | identifier

Stages: ``butter(kind, order, fc)``, ``cheby1(kind, order, fc, ripple_db)``,
``loshelf/hishelf/peak(fc, gain_db[, q])``, ``fir(kind, num_taps, fc=...)``
(band-pass: ``f1=, f2=``; ``window=`` optional). Errors carry the 1-based
column: ``ParseError`` (with the expected tokens), ``UnknownFilter``,
``UnknownArgument``, ``MissingRequiredArgument``; design errors are re-raised
with the offending stage's column span. The parsed Chain runs through the
fused GPU plan like any other.
"""

from __future__ import annotations

import re
from typing import Callable, Dict, List, NamedTuple, Tuple

from .chain import Chain
from .design import design_butterworth, design_chebyshev1, design_fir, design_peaking, design_shelf
from .errors import InvalidArgument, MissingRequiredArgument, ParseError, UnknownArgument, UnknownFilter

__all__ = ["parse_chain_spec", "FILTER_NAMES"]


class _Tok(NamedTuple):
    kind: str  # "number", "name", "|", "(", ")", ",", "=", "end"
    text: str
    col: int   # 1-based


_LEX = re.compile(r"\s+|(-?(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?)|([A-Za-z_]\w*)|([|(),=])")


def _lex(text: str) -> List[_Tok]:
    out, i = [], 0
    while i < len(text):
        m = _LEX.match(text, i)
        if m is None:
            raise ParseError(f"unexpected character {text[i]!r}", i + 1)
        if m.group(1) is not None:
            out.append(_Tok("number", m.group(1), i + 1))
        elif m.group(2) is not None:
            out.append(_Tok("name", m.group(2), i + 1))
        elif m.group(3) is not None:
            out.append(_Tok(m.group(3), m.group(3), i + 1))
        i = m.end()
    out.append(_Tok("end", "", len(text) + 1))
    return out


def _fir(a: Dict):
    kind = a.get("kind", "lowpass")
    if str(kind).lower() in ("bp", "bandpass"):
        missing = [k for k in ("f1", "f2") if k not in a]
        if missing:
            raise MissingRequiredArgument(f"fir bandpass needs {', '.join(missing)}", 0)
        fc = (a["f1"], a["f2"])
    else:
        if "fc" not in a:
            raise MissingRequiredArgument("fir needs fc", 0)
        fc = a["fc"]
    return design_fir(kind, a["num_taps"], fc, a.get("window", "hamming"))


def _q(a: Dict) -> Dict:
    return {"q": a["q"]} if "q" in a else {}


# name -> (positional order, required, optional, builder)
_CATALOG: Dict[str, Tuple[Tuple[str, ...], Tuple[str, ...], Tuple[str, ...], Callable]] = {
    "butter": (("kind", "order", "fc"), ("kind", "order", "fc"), (),
               lambda a: design_butterworth(a["kind"], a["order"], a["fc"])),
    "cheby1": (("kind", "order", "fc", "ripple_db"), ("kind", "order", "fc", "ripple_db"), (),
               lambda a: design_chebyshev1(a["kind"], a["order"], a["ripple_db"], a["fc"])),
    "loshelf": (("fc", "gain_db", "q"), ("fc", "gain_db"), ("q",),
                lambda a: design_shelf("lo_shelf", a["fc"], a["gain_db"], **_q(a))),
    "hishelf": (("fc", "gain_db", "q"), ("fc", "gain_db"), ("q",),
                lambda a: design_shelf("hi_shelf", a["fc"], a["gain_db"], **_q(a))),
    "peak": (("fc", "gain_db", "q"), ("fc", "gain_db"), ("q",),
             lambda a: design_peaking(a["fc"], a["gain_db"], **_q(a))),
    "fir": (("kind", "num_taps"), ("kind", "num_taps"), ("fc", "f1", "f2", "window"), _fir),
}

FILTER_NAMES = tuple(sorted(_CATALOG))


class _Reader:
    def __init__(self, text: str):
        self.toks = _lex(text)
        self.i = 0

    def peek(self, k: int = 0) -> _Tok:
        return self.toks[min(self.i + k, len(self.toks) - 1)]

    def take(self) -> _Tok:
        t = self.toks[self.i]
        self.i += 1
        return t

    def need(self, kind: str, what: str) -> _Tok:
        t = self.peek()
        if t.kind != kind:
            raise ParseError(f"unexpected {t.text or 'end of input'!r}", t.col, expected=(what,))
        return self.take()

    def value(self):
        t = self.peek()
        if t.kind == "number":
            self.take()
            return int(t.text) if re.fullmatch(r"-?\d+", t.text) else float(t.text)
        if t.kind == "name":
            self.take()
            return t.text
        raise ParseError(f"unexpected {t.text or 'end of input'!r}", t.col, expected=("number", "identifier"))

    def args(self, name: str, positional, required, optional) -> Dict:
        out: Dict = {}
        if self.peek().kind == ")":
            return out
        allowed = set(positional) | set(required) | set(optional)
        npos, seen_kw = 0, False
        while True:
            t = self.peek()
            if t.kind == "name" and self.peek(1).kind == "=":
                self.take()
                self.take()
                if t.text not in allowed:
                    raise UnknownArgument(
                        f"{name} does not accept argument {t.text!r} (accepts: {', '.join(sorted(allowed))})", t.col)
                if t.text in out:
                    raise ParseError(f"duplicate argument {t.text!r}", t.col)
                out[t.text] = self.value()
                seen_kw = True
            else:
                if seen_kw:
                    raise ParseError("positional argument after keyword argument", t.col)
                if npos >= len(positional):
                    raise ParseError(f"too many positional arguments for {name}", t.col,
                                     expected=("keyword argument", "')'"))
                if positional[npos] in out:
                    raise ParseError(f"duplicate argument {positional[npos]!r}", t.col)
                out[positional[npos]] = self.value()
                npos += 1
            if self.peek().kind != ",":
                return out
            self.take()

    def stage(self):
        nt = self.need("name", "filter name")
        if nt.text not in _CATALOG:
            raise UnknownFilter(f"unknown filter {nt.text!r} (known: {', '.join(FILTER_NAMES)})", nt.col)
        positional, required, optional, build = _CATALOG[nt.text]
        self.need("(", "'('")
        a = self.args(nt.text, positional, required, optional)
        close = self.need(")", "')'")
        missing = [p for p in required if p not in a]
        if missing:
            raise MissingRequiredArgument(f"{nt.text} is missing required argument(s): {', '.join(missing)}", nt.col)
        try:
            return build(a)
        except MissingRequiredArgument as exc:
            raise type(exc)(str(exc).split(": ", 1)[-1], nt.col) from None
        except InvalidArgument as exc:
            raise type(exc)(f"stage '{nt.text}' (columns {nt.col}-{close.col}): {exc}") from None

    def chain(self) -> Chain:
        stages = [self.stage()]
        while self.peek().kind == "|":
            self.take()
            stages.append(self.stage())
        t = self.peek()
        if t.kind != "end":
            raise ParseError(f"unexpected {t.text!r} after stage", t.col, expected=("'|'", "end of input"))
        return Chain(stages)


def parse_chain_spec(text: str) -> Chain:
    """Parse chain-spec text into an unbound Chain (chainspec.py:236-250)."""
    return _Reader(text).chain()
