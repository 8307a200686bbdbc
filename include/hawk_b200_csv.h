/* hawk_b200_csv.h — CSV ingest into device columns.
 *
 * The reference loads CSV on the host, row by row, into a Table
 * (load_csv, /root/reference/proj/src/storage_csv.cpp:111-155: RFC-4180
 * records, quoted fields with doubled quotes and embedded newlines, an empty
 * line ends the input, int64 via from_chars, float64 via stod, strings
 * dictionary-encoded in first-appearance order by Table::append_row,
 * storage_table.cpp:127-135). Here the file's bytes are copied to HBM once
 * and parsed there: a quote-parity scan finds the record boundaries, one
 * thread parses each record into the int64 / float64 columns, and string
 * fields are hashed and ranked by first appearance on the device. Float
 * fields outside the exactly-representable fast path and files whose quoting
 * the parity scan cannot follow are finished on the host with the same rules.
 */
#ifndef HAWK_B200_CSV_H
#define HAWK_B200_CSV_H

#include <stdint.h>

#include "hawk_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hawk_csv hawk_csv;

/* column kinds, as the reference's ColumnKind (storage/column.hpp) */
enum { HAWK_CSV_INT64 = 0, HAWK_CSV_FLOAT64 = 1, HAWK_CSV_STRING = 2 };

/* Copies `bytes` bytes of CSV text to the device and finds its records.
 * header = 1 skips the first record (CsvOptions::header). */
int32_t hawk_b200_csv_open(hawk_ctx* ctx, const void* text, int64_t bytes, char delimiter,
                           int32_t header, hawk_csv** out);
/* data records (after the header, before the first empty line) */
int64_t hawk_b200_csv_rows(const hawk_csv* csv);
/* Parses every record into ncols device columns d_columns[c] (8 bytes per
 * row: int64, float64 bits, or string codes). On a malformed field returns
 * HAWK_ERR_INVALID_PARAMS with *error_record (0-based data record) and
 * *error_field set and hawk_b200_csv_error() describing it. */
int32_t hawk_b200_csv_parse(hawk_csv* csv, int32_t ncols, const int32_t* kinds,
                            int64_t* const* d_columns, int64_t* error_record, int32_t* error_field);
const char* hawk_b200_csv_error(const hawk_csv* csv);
/* the dictionary of a string column, in code (= first-appearance) order */
int64_t hawk_b200_csv_lexicon_size(const hawk_csv* csv, int32_t column);
const char* hawk_b200_csv_lexicon(const hawk_csv* csv, int32_t column, int64_t code);
/* 1 when the last parse was finished on the host (quoting the parallel scan
 * cannot follow), 0 when it ran on the device */
int32_t hawk_b200_csv_host_parsed(const hawk_csv* csv);
int32_t hawk_b200_csv_close(hawk_csv* csv);

#ifdef __cplusplus
}
#endif

#endif /* HAWK_B200_CSV_H */
