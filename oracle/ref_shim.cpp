// TEST INFRASTRUCTURE ONLY — the parity checker, never the product path.
//
// A thin extern "C" shim over the UNMODIFIED reference oracle so Python tests
// (ctypes) can build reference `hawk::Table`s, run `hawk::reference_execute`
// and compare results with `hawk::compare_result_tables` / `result_checksum`.
// It is compiled together with the reference's own sources, read in place from
// /root/reference/proj/src (see oracle/Makefile); no reference source is copied.
//
// Reference entry points wrapped here:
//   sql::parse_query            /root/reference/proj/src/sql_parser.cpp:785-793
//   sql::make_catalog           /root/reference/proj/src/sql_parser.cpp:809-813
//   reference_execute           /root/reference/proj/src/planner_reference.cpp:331
//   compare_result_tables       /root/reference/proj/src/planner_result.cpp:48-84
//   result_checksum             /root/reference/proj/src/planner_result.cpp:86-112
//   gen_lineorder/part/supplier /root/reference/proj/src/storage_generator.cpp:33-103
//   partition_into_pipelines    /root/reference/proj/src/planner_pipelines.cpp:550-554
//   load_csv                    /root/reference/proj/src/storage_csv.cpp:111-155
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "hawk/error.hpp"
#include "hawk/planner/pipelines.hpp"
#include "hawk/planner/reference.hpp"
#include "hawk/planner/result.hpp"
#include "hawk/sql/parser.hpp"
#include "hawk/storage/csv.hpp"
#include "hawk/storage/generator.hpp"

namespace hawk::cpu_o {
Table execute(const std::string& sql, const std::vector<TablePtr>& tables, int threads);
}

namespace {

struct OraTable {
  hawk::TablePtr table;
};

struct OraDb {
  std::vector<hawk::TablePtr> tables;
};

void put_err(char* buf, int len, const std::string& s) {
  if (!buf || len <= 0) return;
  std::strncpy(buf, s.c_str(), static_cast<std::size_t>(len - 1));
  buf[len - 1] = 0;
}

// Error classes, 1:1 with include/hawk_b200.h HAWK_ERR_* (hawk/error.hpp:9-54).
int classify(const std::exception& e) {
  if (dynamic_cast<const hawk::DuplicateKey*>(&e)) return 6;
  if (dynamic_cast<const hawk::EmptyAggregate*>(&e)) return 7;
  if (dynamic_cast<const hawk::CapacityExceeded*>(&e)) return 5;
  if (dynamic_cast<const hawk::PlanTooLarge*>(&e)) return 4;
  if (dynamic_cast<const hawk::InvalidConfig*>(&e)) return 2;
  if (dynamic_cast<const hawk::Unsupported*>(&e)) return 3;
  if (dynamic_cast<const hawk::UnsupportedPlan*>(&e)) return 1;
  if (dynamic_cast<const hawk::SyntaxError*>(&e)) return 10;
  if (dynamic_cast<const hawk::UnknownTable*>(&e)) return 11;
  if (dynamic_cast<const hawk::UnknownAttribute*>(&e)) return 12;
  if (dynamic_cast<const hawk::TypeError*>(&e)) return 13;
  if (dynamic_cast<const hawk::DivergentPlan*>(&e)) return 8;
  return 99;
}

}  // namespace

extern "C" {

// ---- tables -------------------------------------------------------------

// kinds: 0 = int64, 1 = float64, 2 = string (data = int64 codes into lexicon).
// Rows are appended through Table::append_row, so string columns get the
// reference's first-appearance dictionary order.
OraTable* ora_table_new(const char* name, int ncols, const char* const* names, const int* kinds,
                        int64_t nrows, const void* const* data,
                        const char* const* const* lexicons, const int64_t* lexicon_sizes,
                        char* err, int errlen) {
  try {
    hawk::Schema schema;
    for (int c = 0; c < ncols; ++c)
      schema.push_back({names[c], static_cast<hawk::ColumnKind>(kinds[c])});
    auto t = std::make_shared<hawk::Table>(name, schema);
    hawk::Row row(static_cast<std::size_t>(ncols));
    for (int64_t r = 0; r < nrows; ++r) {
      for (int c = 0; c < ncols; ++c) {
        switch (kinds[c]) {
          case 0: row[c] = static_cast<const int64_t*>(data[c])[r]; break;
          case 1: row[c] = static_cast<const double*>(data[c])[r]; break;
          default: {
            int64_t code = static_cast<const int64_t*>(data[c])[r];
            if (code < 0 || code >= lexicon_sizes[c]) throw hawk::Error("bad string code");
            row[c] = std::string(lexicons[c][code]);
          }
        }
      }
      t->append_row(row);
    }
    t->finalize();
    return new OraTable{t};
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return nullptr;
  }
}

OraTable* ora_table_gen(const char* which, int64_t n, uint64_t seed, char* err, int errlen) {
  try {
    std::string w = which;
    hawk::Table t = w == "lineorder" ? hawk::gen_lineorder(static_cast<std::size_t>(n), seed)
                    : w == "part"    ? hawk::gen_part(static_cast<std::size_t>(n), seed)
                    : w == "supplier"
                        ? hawk::gen_supplier(static_cast<std::size_t>(n), seed)
                        : throw hawk::Error("unknown generator " + w);
    return new OraTable{std::make_shared<hawk::Table>(std::move(t))};
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return nullptr;
  }
}

// the reference's load_csv (storage_csv.cpp:111-155); kinds as ora_table_new
OraTable* ora_table_load_csv(const char* path, const char* name, int ncols, const char* const* names,
                             const int* kinds, char delimiter, int header, char* err, int errlen) {
  try {
    hawk::Schema schema;
    for (int c = 0; c < ncols; ++c) schema.push_back({names[c], static_cast<hawk::ColumnKind>(kinds[c])});
    hawk::CsvOptions opt;
    opt.delimiter = delimiter;
    opt.header = header != 0;
    return new OraTable{std::make_shared<hawk::Table>(hawk::load_csv(path, name, schema, opt))};
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return nullptr;
  }
}

void ora_table_free(OraTable* t) { delete t; }
int64_t ora_table_rows(const OraTable* t) { return static_cast<int64_t>(t->table->row_count()); }
int ora_table_ncols(const OraTable* t) { return static_cast<int>(t->table->column_count()); }
const char* ora_table_name(const OraTable* t) { return t->table->name().c_str(); }
const char* ora_table_col_name(const OraTable* t, int c) {
  return t->table->column_name(static_cast<std::size_t>(c)).c_str();
}
int ora_table_col_kind(const OraTable* t, int c) {
  return static_cast<int>(t->table->column(static_cast<std::size_t>(c)).kind());
}
const void* ora_table_col_data(const OraTable* t, int c) {
  const hawk::Column& col = t->table->column(static_cast<std::size_t>(c));
  if (col.kind() == hawk::ColumnKind::Float64) return col.floats().data();
  return col.ints().data();
}
int64_t ora_table_col_lexicon_size(const OraTable* t, int c) {
  return static_cast<int64_t>(t->table->column(static_cast<std::size_t>(c)).lexicon().size());
}
const char* ora_table_col_lexicon(const OraTable* t, int c, int64_t i) {
  return t->table->column(static_cast<std::size_t>(c)).lexicon()[static_cast<std::size_t>(i)].c_str();
}
int64_t ora_table_col_distinct(const OraTable* t, int c) {
  return static_cast<int64_t>(t->table->column(static_cast<std::size_t>(c)).distinct_count());
}

uint64_t ora_table_checksum(const OraTable* t) { return hawk::result_checksum(*t->table); }

// 0 when equal (canonical multiset, floats within rel_tol); 1 with a diff message.
int ora_compare(const OraTable* expected, const OraTable* actual, double rel_tol, char* msg,
                int msglen) {
  auto diff = hawk::compare_result_tables(*expected->table, *actual->table, rel_tol);
  if (!diff) return 0;
  put_err(msg, msglen, *diff);
  return 1;
}

// ---- databases + oracle execution -----------------------------------------

OraDb* ora_db_new() { return new OraDb; }
void ora_db_free(OraDb* db) { delete db; }
void ora_db_add(OraDb* db, const OraTable* t) { db->tables.push_back(t->table); }

// Runs the reference oracle. Returns nullptr on error; *err_class gets the
// hawk error class (see classify) and err the message.
OraTable* ora_execute(OraDb* db, const char* sql, int* err_class, char* err, int errlen) {
  try {
    auto plan = hawk::sql::parse_query(sql, hawk::sql::make_catalog(db->tables));
    hawk::Table out = hawk::reference_execute(plan, db->tables);
    *err_class = 0;
    return new OraTable{std::make_shared<hawk::Table>(std::move(out))};
  } catch (const std::exception& e) {
    *err_class = classify(e);
    put_err(err, errlen, e.what());
    return nullptr;
  }
}

// The reference's CPU variant "cpu-o" over the reference pipeline programs
// (oracle/cpu_o.cpp); same error convention as ora_execute.
OraTable* ora_execute_cpu_o(OraDb* db, const char* sql, int threads, int* err_class, char* err, int errlen) {
  try {
    hawk::Table out = hawk::cpu_o::execute(sql, db->tables, threads);
    *err_class = 0;
    return new OraTable{std::make_shared<hawk::Table>(std::move(out))};
  } catch (const std::exception& e) {
    *err_class = classify(e);
    put_err(err, errlen, e.what());
    return nullptr;
  }
}

// Number of pipelines the reference lowering produces (structure checks).
int ora_pipeline_count(OraDb* db, const char* sql, char* err, int errlen) {
  try {
    auto plan = hawk::sql::parse_query(sql, hawk::sql::make_catalog(db->tables));
    auto set = hawk::partition_into_pipelines(plan, db->tables);
    return static_cast<int>(set.pipelines.size());
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return -1;
  }
}

}  // extern "C"
